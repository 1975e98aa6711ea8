"""Per-step latency of k_exact on a small (L2-resident) index: time of one
launch over 10,000 present patterns as a function of the pattern length.

    python tools/exact_latency.py [n_bases]
"""
import ctypes as ct
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.Generator(np.random.PCG64(42))
text = rng.integers(0, 4, n, dtype=np.uint8)
idx = fm.build_index(text)
dix = idx.device_index(0)
lib = _lib.load()
st = torch.cuda.Stream()
for count in tuple(int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['10000', '100000'])):
    for m in (13, 16, 20, 24, 28, 32):
        pats = workloads.substrings(text, rng.integers(0, n - m + 1, count), m)
        packed = fm.pack_patterns_u64(pats)
        d_pat = torch.from_numpy(packed.view(np.int64)).cuda()
        d_out = torch.empty((count, 2), dtype=torch.int32, device="cuda")
        args = (dix.handle, d_pat.data_ptr(), m, count, d_out.data_ptr(), st.cuda_stream)
        for _ in range(5):
            lib.fmg_exact_packed(*args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(reps):
                lib.fmg_exact_packed(*args)
            e1.record(st)
        torch.cuda.synchronize()
        print(f"count {count} m {m}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per launch", flush=True)
