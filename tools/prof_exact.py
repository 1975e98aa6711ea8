"""Exact-search throughput on config 4 (2^28 x 20 bp seeds, 1 Gbp) and parity on a sample.

usage: python tools/prof_exact.py [count_log2] [reps]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402

count = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 28)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
wl = workloads.config4(count=count)
t1 = time.time()
idx = fm.build_index(wl.text, builder="gpu")
t2 = time.time()
print(f"gen {t1 - t0:.1f}s build {t2 - t1:.1f}s", flush=True)
lib = _lib.load()
dix = idx.device_index(0)
d_pat = torch.from_numpy(wl.packed.view(np.int64)).cuda()
d_out = torch.empty((count, 2), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for r in range(reps + 1):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    _lib.check(lib.fmg_exact_packed(dix.handle, d_pat.data_ptr(), 20, count, d_out.data_ptr(), s))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {r}: {ms:.2f} ms, {count / ms / 1e6:.3f} G seeds/s", flush=True)
kl = d_out.cpu().numpy().view(np.uint32).astype(np.int64)
sample = workloads.unpack_patterns(wl.packed[: 1 << 20], 20)
want = orc.exact_batch(orc.OracleIndex(idx), sample)
print("parity first 2^20 vs oracle:", np.array_equal(kl[: 1 << 20], want))
width = np.maximum(kl[:, 1] - kl[:, 0] + 1, 0)
print("hit fraction", float((width > 0).mean()), "mean width of hits", float(width[width > 0].mean()))
