"""Minimal k_occ_pair driver for ncu: `python tools/prof_occ.py [config1|synthetic_1G] [granularity]`.

Launches: 3 warm-up + 2 measured launches of 2^24 pairs (pass -s 3 -c 1 to ncu).
"""
import ctypes as ct
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402
from sweep_occ import synthetic_index  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "config1"
gran = int(sys.argv[2]) if len(sys.argv) > 2 else -1
lib = _lib.load()
lib.fmgx_set_l2_fetch_granularity.argtypes = [ct.c_int, ct.c_int, ct.POINTER(ct.c_int)]
torch.cuda.init()
prev = ct.c_int()
_lib.check(lib.fmgx_set_l2_fetch_granularity(0, gran, ct.byref(prev)))
print("l2 fetch granularity: previous", prev.value, "now", gran)
if which == "config1":
    idx, n = fm.build_index(workloads.config1().text), 1 << 24
elif which == "config1h":
    wl = workloads.config1h()
    idx, n = fm.build_index(wl.text, builder="gpu"), wl.text.size
elif which == "synthetic_3G":
    idx, n = synthetic_index(3_000_000_000), 3_000_000_000
else:
    idx, n = synthetic_index(1_000_000_000), 1_000_000_000
pairs = wl.pairs if which == "config1h" else workloads.occ_pairs(n, 1 << 24, (7, 1))
kl = np.stack([pairs[:, 0] + 1, pairs[:, 1]], 1).astype(np.uint32)
d_kl = torch.from_numpy(kl.view(np.int32)).cuda()
d_out = torch.empty((kl.shape[0], 8), dtype=torch.int32, device="cuda")
h = idx.device_index(0).handle
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for i in range(5):
    if i == 3:
        e0.record()
    _lib.check(lib.fmg_occ_pair(h, d_kl.data_ptr(), kl.shape[0], d_out.data_ptr(), None, s))
e1.record()
torch.cuda.synchronize()
print(which, "us/launch", e0.elapsed_time(e1) / 2 * 1e3)
