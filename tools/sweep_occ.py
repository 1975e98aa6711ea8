"""Tuning sweep for k_occ_pair: pairs/thread x block size, L2-resident and HBM-resident indexes.

The HBM-resident case uses a synthetic 1 Gbp index (random packed lines) —
valid for timing only, since the kernel's memory behaviour does not depend
on whether the lines hold a real BWT.  Parity is covered by tests/.
"""
import ctypes as ct
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402
from bench import occ_step_bytes  # noqa: E402


def synthetic_index(n: int) -> fm.FmIndex:
    nb = (n + 1 + 127) // 128
    rng = np.random.Generator(np.random.PCG64(5))
    rec = np.zeros((nb, 64), dtype=np.uint8)
    rec[:, 32:] = rng.integers(0, 256, (nb, 32), dtype=np.uint8)
    c = [0, n // 4, n // 2, 3 * n // 4, n]
    return fm.FmIndex(n, c, rec, 0, np.zeros(n // 32 + 1, np.uint64), [fm.RecordSpan("ref", 0, n)])


def main():
    lib = _lib.load()
    fn = lib.fmgx_occ_pair_tuned
    fn.argtypes = [ct.c_void_p] * 2 + [ct.c_uint64, ct.c_void_p, ct.c_void_p, ct.c_int, ct.c_int]
    dev = torch.device("cuda:0")
    out = {}
    cases = [("config1", fm.build_index(workloads.config1().text), 1 << 24)]
    if "--big" in sys.argv:
        cases.append(("synthetic_1G", synthetic_index(1_000_000_000), 1_000_000_000))
    for name, idx, n in cases:
        pairs = workloads.occ_pairs(n, 1 << 24, (7, 1))
        alg, _ = occ_step_bytes(pairs)
        kl = np.stack([pairs[:, 0] + 1, pairs[:, 1]], 1).astype(np.uint32)
        d_kl = torch.from_numpy(kl.view(np.int32)).to(dev)
        d_out = torch.empty((kl.shape[0], 8), dtype=torch.int32, device=dev)
        h = idx.device_index(0).handle
        s = torch.cuda.current_stream().cuda_stream
        for per in (1, 2):
            for threads in (64, 128, 256):
                for _ in range(3):
                    _lib.check(fn(h, d_kl.data_ptr(), kl.shape[0], d_out.data_ptr(), s, per, threads))
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(20):
                    fn(h, d_kl.data_ptr(), kl.shape[0], d_out.data_ptr(), s, per, threads)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 20 / 1e3
                out[f"{name}/per{per}/t{threads}"] = {"us": round(t * 1e6, 1), "Gsteps_s": round(kl.shape[0] / t / 1e9, 2),
                                                     "alg_GBs": round(alg / t / 1e9, 1)}
                print(name, per, threads, out[f"{name}/per{per}/t{threads}"], flush=True)
        idx.release_device()
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/sweep_occ.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
