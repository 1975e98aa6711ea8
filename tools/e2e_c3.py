"""Where the config-3 end-to-end step spends its time (host entry points, pinned buffers).

usage: python tools/e2e_c3.py [n_reads]   -- per-call wall times of the exact pass, every z=1 chunk and its copy-out
"""
import ctypes as ct
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import PinnedResults  # noqa: E402

n_reads = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
wl = workloads.config3(n_reads=n_reads)
idx = fm.build_index(wl.text, builder="gpu")
lib = _lib.load()
dix = idx.device_index(0)
n_seeds = wl.packed.size
pin_in = torch.from_numpy(wl.packed.view(np.int64)).pin_memory()
pin_kl = torch.empty((n_seeds, 2), dtype=torch.int32).pin_memory()
host_res = PinnedResults()
copier = ThreadPoolExecutor(max_workers=1)
chunk = -(-n_seeds // max(1, -(-n_seeds // (1 << 24))))
chunk = min(chunk, 14_000_000)


def copy_out(h, cnt, log):
    t = time.perf_counter()
    try:
        return host_res.copy(lib, h, cnt)
    finally:
        t1 = time.perf_counter()
        lib.fmg_matches_free(h)
        log.append((1e3 * (t1 - t), 1e3 * (time.perf_counter() - t1)))


for rep in range(4):
    t0 = time.perf_counter()
    _lib.check(lib.fmg_exact_packed_host(dix.handle, pin_in.data_ptr(), 19, n_seeds, pin_kl.data_ptr()))
    t1 = time.perf_counter()
    calls, copies, pending = [], [], []
    for c0 in range(0, n_seeds, chunk):
        cnt = min(chunk, n_seeds - c0)
        h = ct.c_void_p()
        ta = time.perf_counter()
        _lib.check(lib.fmg_inexact_packed_host(dix.handle, pin_in.data_ptr() + 8 * c0, 19, cnt, 1, ct.byref(h)))
        calls.append(1e3 * (time.perf_counter() - ta))
        pending.append(copier.submit(copy_out, h, cnt, copies))
    t2 = time.perf_counter()
    nbytes = sum(f.result() for f in pending)
    t3 = time.perf_counter()
    print(f"rep {rep}: exact {1e3 * (t1 - t0):.1f} ms, z=1 calls {[round(c, 1) for c in calls]} ms (sum {sum(calls):.1f}), "
          f"copies (copy, free) {[(round(a, 1), round(b, 1)) for a, b in copies]}, wait for last copy {1e3 * (t3 - t2):.1f} ms, "
          f"total {1e3 * (t3 - t0):.1f} ms, {nbytes / 1e9:.2f} GB out -> {n_reads / (t3 - t0) / 1e6:.2f} M reads/s", flush=True)
