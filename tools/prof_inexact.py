"""Drive fmg_inexact on config 2 (device-resident seeds) for timing / ncu.

usage: python tools/prof_inexact.py [n_reads] [reps]
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
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = _lib.load()
wl = workloads.config2(n_reads=n_reads)
idx = fm.build_index(wl.text)
dix = idx.device_index(0)
if int(__import__("os").environ.get("FMG_BIDIR", "0")):
    dix.ensure_reverse()
m = wl.patterns.shape[1]
codes = np.ascontiguousarray(wl.patterns.reshape(-1))
offs = np.arange(0, (n_reads + 1) * m, m, dtype=np.uint64)
d_codes = torch.from_numpy(codes).cuda()
d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
s = torch.cuda.Stream()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = ct.c_void_p()
    _lib.check(lib.fmg_inexact(dix.handle, d_codes.data_ptr(), d_offs.data_ptr(), n_reads, 1, ct.byref(h),
                               s.cuda_stream))
    t1 = time.perf_counter()
    tot, steps = ct.c_uint64(), ct.c_uint64()
    lib.fmg_matches_size(h, ct.byref(tot), None)
    lib.fmg_matches_steps(h, ct.byref(steps))
    lib.fmg_matches_free(h)
    t2 = time.perf_counter()
    print(f"rep {r}: inexact {1e3 * (t1 - t0):.1f} ms, free {1e3 * (t2 - t1):.1f} ms, results {tot.value}, "
          f"steps {steps.value} ({steps.value / n_reads:.1f}/read), {n_reads / (t1 - t0) / 1e6:.2f} M reads/s",
          flush=True)
