"""Config-3 style inexact z=1 timing at genome scale with fewer reads (engine A/B).

usage: python tools/prof_c3.py [n_reads] [reps]   (FMG_INEXACT_DFS / FMG_LIB_PATH / FMG_TRACE honoured)
"""
import ctypes as ct
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402

n_reads = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
wl = workloads.config3(n_reads=n_reads)
idx = fm.build_index(wl.text, builder="gpu")
print(f"gen+build {time.time() - t0:.1f}s, seeds {wl.packed.size}", flush=True)
lib = _lib.load()
dix = idx.device_index(0)
if int(__import__("os").environ.get("FMG_BIDIR", "1")) and dix.wants_reverse(wl.packed.size, 19, 1):
    t3 = time.time()
    dix.ensure_reverse()
    print(f"reverse index {time.time() - t3:.1f}s", flush=True)
d = torch.from_numpy(wl.packed.view(np.int64)).cuda()
s = torch.cuda.Stream()
times = []
for r in range(reps):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = ct.c_void_p()
    _lib.check(lib.fmg_inexact_packed(dix.handle, d.data_ptr(), 19, wl.packed.size, 1, ct.byref(h), s.cuda_stream))
    t2 = time.perf_counter()
    tot, steps, lines = ct.c_uint64(), ct.c_uint64(), ct.c_uint64()
    lib.fmg_matches_size(h, ct.byref(tot), None)
    lib.fmg_matches_steps(h, ct.byref(steps))
    lib.fmgx_matches_lines(h, ct.byref(lines))
    kk = np.empty(tot.value, np.uint32)
    dd = np.empty(tot.value, np.uint8)
    row = np.empty(wl.packed.size + 1, np.uint64)
    lib.fmg_matches_copy(h, row.ctypes.data, kk.ctypes.data, None, dd.ctypes.data, 1)
    lib.fmg_matches_free(h)
    times.append(t2 - t1)
    print(f"rep {r}: {1e3 * (t2 - t1):.1f} ms, {wl.packed.size / (t2 - t1) / 1e6:.2f} M seeds/s, results {tot.value}, "
          f"steps/seed {steps.value / wl.packed.size:.0f}, lines/seed {lines.value / wl.packed.size:.0f}, "
          f"checksum {int(kk.astype(np.uint64).sum()) ^ int(row.sum()) ^ int(dd.sum())}", flush=True)
ts = sorted(times[1:] or times)
print(f"summary: median {1e3 * ts[len(ts) // 2]:.1f} ms, min {1e3 * ts[0]:.1f} ms over {len(ts)} reps after the first",
      flush=True)
