"""Per-call wall time of fmg_inexact on config 2 (z = 1), device inputs, on
several stream kinds; with FMG_TRACE=1 the library prints its phase times.

    python tools/time_c2.py [--reads N]
"""
import argparse
import ctypes as ct
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1811_06127_b200 as fm  # noqa: E402
from paper_1811_06127_b200 import _lib, workloads as w  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reads", type=int, default=1_000_000)
ap.add_argument("--reverse", type=int, default=1)
args = ap.parse_args()
wl = w.config2(n_reads=args.reads)
idx = fm.build_index(wl.text)
dix = idx.device_index(0)
if args.reverse:
    dix.ensure_reverse()
lib = _lib.load()
units, m = wl.patterns.shape
codes = np.ascontiguousarray(wl.patterns.reshape(-1))
offs = np.arange(0, (units + 1) * m, m, dtype=np.uint64)
dev = torch.device("cuda:0")
d_codes = torch.from_numpy(codes).to(dev)
d_offs = torch.from_numpy(offs.view(np.int64)).to(dev)
import subprocess
smi = None
for kind in ("torch", "null", "torch+smi", "null+smi"):
    if kind.endswith("+smi") and smi is None:
        smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap",
                                "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    st = torch.cuda.Stream(dev) if kind.startswith("torch") else None
    sp = st.cuda_stream if st is not None else 0
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = ct.c_void_p()
        _lib.check(lib.fmg_inexact(dix.handle, d_codes.data_ptr(), d_offs.data_ptr(), units, 1, ct.byref(h),
                                   ct.c_void_p(sp)))
        t1 = time.perf_counter()
        lib.fmg_matches_free(h)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ts.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2)))
    print(kind, "call ms / free+sync ms:", ts, flush=True)
if smi is not None:
    smi.terminate()
# back to back without host syncs between calls, CUDA events on the stream (bench.py's loop)
for prefix in (0, 1):
    if prefix:
        fn = lib.fmgx_prefix_table
        fn.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint64)]
        kk, nb = ct.c_uint32(), ct.c_uint64()
        _lib.check(fn(dix.handle, ct.byref(kk), ct.byref(nb)))
    for kind in ("torch", "null"):
        st = torch.cuda.Stream(dev) if kind == "torch" else torch.cuda.default_stream(dev)
        torch.cuda.set_stream(st)
        sp = st.cuda_stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(10):
            h = ct.c_void_p()
            _lib.check(lib.fmg_inexact(dix.handle, d_codes.data_ptr(), d_offs.data_ptr(), units, 1, ct.byref(h),
                                       ct.c_void_p(sp)))
            lib.fmg_matches_free(h)
        e1.record(st)
        torch.cuda.synchronize()
        print("prefix", prefix, kind, "back-to-back ms/call", e0.elapsed_time(e1) / 10, flush=True)
