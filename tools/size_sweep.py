"""k_occ_pair throughput vs index size (synthetic indexes; timing only)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402
from sweep_occ import synthetic_index  # noqa: E402
from bench import occ_step_bytes  # noqa: E402

lib = _lib.load()
for n in [1 << 24, 1 << 26, 1 << 27, 1 << 28, 1 << 29, 1 << 30, 3_000_000_000]:
    idx = synthetic_index(n)
    pairs = workloads.occ_pairs(n, 1 << 24, (7, 1))
    alg, _ = occ_step_bytes(pairs)
    kl = np.stack([pairs[:, 0] + 1, pairs[:, 1]], 1).astype(np.uint32)
    d_kl = torch.from_numpy(kl.view(np.int32)).cuda()
    d_out = torch.empty((kl.shape[0], 8), dtype=torch.int32, device="cuda")
    h = idx.device_index(0).handle
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.fmg_occ_pair(h, d_kl.data_ptr(), kl.shape[0], d_out.data_ptr(), None, s)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        lib.fmg_occ_pair(h, d_kl.data_ptr(), kl.shape[0], d_out.data_ptr(), None, s)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 / 1e3
    print(f"n={n:>11d} index={n/2/1e6:8.1f} MB  {kl.shape[0]/t/1e9:6.2f} G steps/s  alg {alg/t/1e9:7.1f} GB/s", flush=True)
    idx.release_device()
    del d_kl, d_out
