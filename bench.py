"""Benchmark: Occ steps/s on BASELINE.json config 1 (default), plus other configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config1]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port)

One step = one pass of the hot path over one batch of synthetic input:
  config1  : fmg_occ_pair over 2^24 (k-1, l) pairs on a 2^24-base index
  config1h : the same pair distribution over the 1 Gbp config-4 text
  config0  : exact search of 10,000 x 32 bp patterns on 1 Mbp
  config2  : inexact (z=1) search of 1,000,000 32-bp seeds on the 64 Mbp repeat genome
  config4  : exact search of 2^28 x 20 bp seeds on 1 Gbp (host memory heavy)
Inputs are resident in HBM when the timed region starts (`value`); `e2e` is
the same metric through the C-ABI host entry point with host buffers and the
host<->device copies inside the timed region.  Multi-GPU: weak scaling, rank
r processes its own shard of the same size; no collective on the data path.
"""

from __future__ import annotations

import argparse
import ctypes as ct
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

PEAKS = REPO / "MEASURED_PEAKS.json"
TRAFFIC = REPO / "profiles" / "traffic.json"


def hbm_peak() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(kernel: str, config: str):
    """dram bytes/launch from the committed ncu --set full capture (profiles/traffic.json)."""
    try:
        return json.loads(TRAFFIC.read_text())[config][kernel]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("FMG_BENCH_CLOCK_MS", "100")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def occ_step_bytes(pairs: np.ndarray) -> tuple[int, int]:
    """Algorithmic bytes of config-1 Occ steps on the line layout.

    Per step: 32 B x |lines(k-1) U lines(l)| + 8 B (k, l) in + 32 B (8 x u32) out.
    Returns (total bytes, total distinct lines).
    """
    low, high = pairs[:, 0], pairs[:, 1]
    two = (low >= 0) & ((low >> 6) != (high >> 6))
    lines = int(low.size + two.sum())
    return lines * 32 + low.size * 40, lines


CHUNK_CHARS = {2: 192, 4: 416}  # sectors per chunk -> characters (csrc/kernels_chunk.cuh)


def chunk_sector_of(r: np.ndarray) -> np.ndarray:
    return np.where(r < 80, 0, 1 + (r - 80) // 112)


def chunk_step_bytes(pairs: np.ndarray, chars: int = 416) -> tuple[int, int, int]:
    """Algorithmic bytes of Occ steps on the 128-byte chunk layout (kernels_chunk.cuh).

    Per step: 32 B x |S(k-1) U S(l)| with S(p) = {sector 0 of p's chunk, the
    sector holding p} + 8 B (k, l) in + 32 B out.  Returns (total bytes,
    total distinct sectors, total distinct chunks)."""
    low, high = pairs[:, 0], pairs[:, 1]
    jh, jl = high // chars, np.maximum(low, 0) // chars
    sh = chunk_sector_of(high - jh * chars)
    sl = chunk_sector_of(np.maximum(low, 0) - jl * chars)
    has_low = low >= 0
    other = has_low & (jl != jh)
    sect = 1 + (sh != 0)                                       # high end: base + its sector
    sect = sect + np.where(other, 1 + (sl != 0), 0)            # low end in another chunk
    sect = sect + (has_low & ~other & (sl != 0) & (sl != sh))  # low end in another sector of the same chunk
    sectors = int(sect.sum())
    chunks = int(low.size + other.sum())
    return sectors * 32 + low.size * 40, sectors, chunks


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class PinnedResults:
    """Reusable pinned host buffers for CSR result sets (row offsets, k, l, diffs).

    The e2e leg copies every step's results to the host like a user
    streaming batches would: into buffers allocated once (grown on demand
    during the untimed first call), not into fresh pageable arrays whose
    first-touch page faults would dominate the copy."""

    def __init__(self):
        import torch

        self.torch = torch
        self.cap_rows = self.cap = 0

    def copy(self, lib, h, patterns: int) -> int:
        tot = ct.c_uint64()
        lib.fmg_matches_size(h, ct.byref(tot), None)
        n = tot.value
        t = self.torch
        if patterns + 1 > self.cap_rows:
            self.cap_rows = patterns + 1
            self.row = t.empty(self.cap_rows, dtype=t.int64).pin_memory()
        if n > self.cap:
            self.cap = max(n, int(self.cap * 1.25))
            self.k = t.empty(self.cap, dtype=t.int32).pin_memory()
            self.l = t.empty(self.cap, dtype=t.int32).pin_memory()
            self.d = t.empty(self.cap, dtype=t.uint8).pin_memory()
        lib.fmg_matches_copy(h, self.row.data_ptr(), self.k.data_ptr(), self.l.data_ptr(), self.d.data_ptr(), 1)
        return (patterns + 1) * 8 + n * 9


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def make_workload(config: str, rank: int):
    from paper_1811_06127_b200 import workloads as w

    if config == "config1":
        return w.config1(shard=rank)
    if config == "config1h":
        return w.config1h()
    if config == "config0":
        return w.config0()
    if config == "config2":
        return w.config2()
    if config == "config4":
        return w.config4()
    if config == "config3":
        return w.config3(n_reads=int(os.environ.get("FMG_C3_READS", 10_000_000)),
                         n=int(os.environ.get("FMG_C3_BASES", 3_100_000_000)))
    raise SystemExit(f"unknown config {config}")


# ---------------------------------------------------------------------------
# multi-rank plumbing: one shared workload, self-launch, result digests
# ---------------------------------------------------------------------------

SHM = Path(os.environ.get("FMG_SHM_DIR", "/dev/shm"))


def shared_workload(config: str, rank: int, world: int, barrier):
    """The workload of `config`, generated ONCE per node: rank 0 writes its
    arrays under /dev/shm, the other ranks memory-map them after the barrier
    (config 3 is a 3.1 Gbp text plus 140M packed seeds: generating it on
    every rank would cost N x the host memory and CPU).  Config 1 draws an
    independent pair set per rank (weak scaling) and is generated locally."""
    from paper_1811_06127_b200.workloads import Workload

    if world == 1 or config == "config1":
        return make_workload(config, rank)
    key = f"{config}_{os.environ.get('FMG_C3_READS', '')}_{os.environ.get('FMG_C3_BASES', '')}"
    d = SHM / f"fmg_wl_{key}_{os.environ.get('MASTER_PORT', '0')}"
    fields = ("text", "patterns", "packed", "pairs")
    if rank == 0:
        wl = make_workload(config, 0)
        d.mkdir(parents=True, exist_ok=True)
        for f in fields:
            a = getattr(wl, f)
            if a is not None:
                np.save(d / f"{f}.npy", a)
        (d / "meta.json").write_text(json.dumps({"name": wl.name, "max_diff": wl.max_diff, "meta": wl.meta}))
    barrier()
    if rank != 0:
        m = json.loads((d / "meta.json").read_text())
        # the text is only read (by the index build): memory-mapped; query arrays are copied in
        arrs = {f: (np.load(d / f"{f}.npy", mmap_mode="r" if f == "text" else None)
                    if (d / f"{f}.npy").exists() else None) for f in fields}
        wl = Workload(m["name"], arrs["text"], patterns=arrs["patterns"], packed=arrs["packed"],
                      pairs=arrs["pairs"], max_diff=m["max_diff"], meta=m["meta"])
    barrier()  # every rank has mapped the arrays: the files can go (the mappings stay valid)
    if rank == 0:
        for f in d.glob("*"):
            f.unlink()
        d.rmdir()
    return wl


def self_launch(args) -> None:
    """`bench.py --gpus N` without a torchrun environment: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def sha_update(h, *arrays) -> None:
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())


def digest_pairs(fm, idx, pairs) -> str:
    import hashlib

    h = hashlib.sha256()
    for c0 in range(0, pairs.shape[0], 1 << 22):
        sha_update(h, fm.occ_pair_batch(idx, pairs[c0:c0 + (1 << 22), 0], pairs[c0:c0 + (1 << 22), 1]))
    return h.hexdigest()


def digest_patterns(lib, dix, wl, lo: int, hi: int) -> str:
    """SHA-256 over exact intervals (and z = 1 result counts / k / l / diffs for
    inexact workloads) of patterns [lo, hi), in chunks of 2^22 patterns."""
    import hashlib

    from paper_1811_06127_b200 import _lib

    h = hashlib.sha256()
    m = wl.meta["m"] if wl.packed is not None else wl.patterns.shape[1]
    step = 1 << 22
    for c0 in range(lo, hi, step):
        c1 = min(hi, c0 + step)
        if wl.packed is not None:
            packed = np.ascontiguousarray(wl.packed[c0:c1])
        else:
            from paper_1811_06127_b200 import pack_patterns_u64

            packed = pack_patterns_u64(np.ascontiguousarray(wl.patterns[c0:c1]))
        if wl.max_diff == 0 or wl.name == "config3":
            kl = np.empty((c1 - c0, 2), dtype=np.uint32)
            _lib.check(lib.fmg_exact_packed_host(dix.handle, packed.ctypes.data, m, c1 - c0, kl.ctypes.data))
            sha_update(h, kl)
        if wl.max_diff:
            hd = ct.c_void_p()
            _lib.check(lib.fmg_inexact_packed_host(dix.handle, packed.ctypes.data, m, c1 - c0, wl.max_diff,
                                                   ct.byref(hd)))
            try:
                tot = ct.c_uint64()
                lib.fmg_matches_size(hd, ct.byref(tot), None)
                row = np.empty(c1 - c0 + 1, dtype=np.uint64)
                k = np.empty(tot.value, dtype=np.uint32)
                l_ = np.empty(tot.value, dtype=np.uint32)
                d = np.empty(tot.value, dtype=np.uint8)
                _lib.check(lib.fmg_matches_copy(hd, row.ctypes.data, k.ctypes.data, l_.ctypes.data, d.ctypes.data, 1))
            finally:
                lib.fmg_matches_free(hd)
            sha_update(h, np.diff(row.astype(np.int64)), k, l_, d)
    return h.hexdigest()


def unit_count(wl) -> int:
    if wl.name == "config3":
        return wl.meta["reads"]
    if wl.pairs is not None:
        return wl.pairs.shape[0]
    return wl.packed.shape[0] if wl.packed is not None else wl.patterns.shape[0]


def pattern_sample(wl, lo: int, hi: int) -> np.ndarray:
    """(hi-lo, m) uint8 codes of a slice of a pattern workload."""
    if wl.packed is not None:
        from paper_1811_06127_b200.workloads import unpack_patterns

        return unpack_patterns(wl.packed[lo:hi], wl.meta["m"])
    return wl.patterns[lo:hi]


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path (oracle port, all host threads)
# ---------------------------------------------------------------------------


# Per-step unit counts of the reference arm: the full workload wherever the
# reference path finishes one step in a few seconds on the box's host cores
# (configs 0, 1, 1-H, 2), a bounded leading sample elsewhere (configs 3, 4).
REF_FULL = {"config0", "config1", "config1h", "config2"}
REF_SAMPLE = {"config4": 1 << 22, "config3": 2_000}


def mem_available() -> int:
    try:
        for ln in Path("/proc/meminfo").read_text().splitlines():
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def native_libs_mapped() -> list[str]:
    """Shared objects of this repo mapped into the current process."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps if ln.endswith(".so") and str(REPO) in ln})


def run_reference(args, rank: int, world: int) -> None:
    """The reference's CPU path on the box's host cores: the index is built by
    the oracle's restatement of build_suffix_array / bwt_from_sa / build_index
    (oracle/fm_build.c) and queried by the restatement of the reference's
    occ_pair_all / exact_search / inexact_search (oracle/fm_oracle.c).  The
    product library (libfmgpu.so) is never loaded in this process."""
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_1811_06127_b200 import workloads as w  # numpy-only generators

    wl = make_workload(args.config, 0)
    threads = cpu_threads()
    need = 14 * wl.text.size  # fm_build.c: sa + rank + key (u32) + records + samples
    avail = mem_available()
    if avail and need > 0.8 * avail:
        print(json.dumps({"impl": "reference", "unavailable": f"the oracle's index build needs ~{need >> 30} GiB, "
                          f"{avail >> 30} GiB available on this host"}), flush=True)
        return
    t_build = time.perf_counter()
    ox = orc.OracleIndex(orc.BuiltIndex(wl.text, threads))
    t_build = time.perf_counter() - t_build
    total = unit_count(wl)
    sample = total if args.config in REF_FULL else min(total, REF_SAMPLE[args.config])
    if args.ref_sample:
        sample = min(total, args.ref_sample)
    if wl.pairs is not None:
        low = np.ascontiguousarray(wl.pairs[:, 0])
        high = np.ascontiguousarray(wl.pairs[:, 1])
    elif wl.name == "config3":
        per = wl.meta["seeds_per_read"]
        seeds3 = pattern_sample(wl, 0, sample * per)
    else:
        pats = pattern_sample(wl, 0, sample)

    def step(i: int):
        if wl.name == "config3":  # reads -> their 14 seeds: exact + z=1
            orc.exact_batch(ox, seeds3, threads)
            orc.inexact_batch(ox, seeds3, 1, threads)
        elif wl.pairs is not None:
            orc.occ_pair_batch(ox, low[:sample], high[:sample], threads)
        elif wl.max_diff:
            orc.inexact_batch(ox, pats, wl.max_diff, threads)
        else:
            orc.exact_batch(ox, pats, threads)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    metric, unit = metric_of(args.config)
    value = sample * args.steps / dt
    what = "the full workload" if sample == total else f"the first {sample} of {total} units"
    desc = (f"C restatement of the reference path (oracle/fm_oracle.c: bytelut all4, occ_pair_all, "
            f"exact/inexact_search; index by oracle/fm_build.c) on {threads} threads of {cpu_model()}; "
            f"{what} per step")
    mapped = native_libs_mapped()
    if any("libfmgpu" in m for m in mapped):
        raise SystemExit("reference arm: the product library was loaded")
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "u32",
        "data": DATA, "config": config_of(args.config, world, total),
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "index_build_s": round(t_build, 2), "units_timed_per_step": sample,
        "native_libs": mapped,
    }
    print(json.dumps(line), flush=True)


DATA = "synthetic (seeded PCG64 per BASELINE.json config; workloads.py)"


def scaling_of(config: str) -> str:
    return "strong" if config in ("config3", "config4") else "weak"


def metric_of(config: str) -> tuple[str, str]:
    if config in ("config1", "config1h"):
        return "Occ steps/sec (8 counts each)", "occ_steps/s"
    return "reads/sec", "reads/s"  # config 3: reads whose 14 seeds got exact + z=1 search


def config_of(config: str, world: int, units: int) -> dict:
    desc = {
        "config1": "BASELINE configs[1]: Occ microbenchmark, 2^24-base iid text (seed 7), 2^24 (k-1,l) pairs/rank",
        "config1h": "config 1-H: config-1 pair distribution over the 1 Gbp config-4 text (HBM-resident index)",
        "config0": "BASELINE configs[0]: exact search, 1 Mbp iid (seed 42), 10,000 x 32 bp",
        "config2": "BASELINE configs[2]: inexact z=1, 64 Mbp repeat genome (seed 3), 1M x 32 bp seeds",
        "config4": "BASELINE configs[4]: exact, 1 Gbp iid (seed 5), 2^28 x 20 bp seeds",
        "config3": "BASELINE configs[3]: 3.1 Gbp family genome (seed 11), 10M x 150 bp reads, 14 x 19 bp seeds "
                   "per read, exact + z=1 on every seed",
    }[config]
    l2 = {
        "config1": "no flush: the 640 MiB of pairs in + counts out per step exceed L2; the 8.4 MB index is "
                   "L2-resident by design (the roofline is the L2 random-read ceiling)",
        "config1h": "no flush: pairs + counts (640 MiB) and the 308 MB chunk layout of the index exceed L2",
        "config0": "inputs smaller than L2; the 1 Mbp index is L2-resident",
        "config2": "no flush: the 32 MB index lines are L2-resident, patterns + results stream",
        "config3": "no flush: the 3.1 Gbp index (1.55 GB of lines) and 140M seeds exceed L2",
        "config4": "no flush: the 1 Gbp index (500 MB of lines) and 2^28 seeds exceed L2",
    }[config]
    return {"workload": desc, "units_per_step_per_rank": units, "parallelism": f"query-sharded x{world}", "l2": l2}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def dist_sum(value: float, world: int, device) -> float:
    """Sum of a per-rank count over all ranks (plumbing only, off the timed path)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def exact_work(lib, dix, d_pat, m: int, count: int, d_out, stream) -> tuple[int, int]:
    """(Occ steps, lines fetched) of one packed exact search, counted on the device."""
    fn = lib.fmgx_exact_packed_work
    fn.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_uint32, ct.c_uint64, ct.c_void_p, ct.c_void_p,
                   ct.POINTER(ct.c_uint64), ct.POINTER(ct.c_uint64)]
    st, ln = ct.c_uint64(), ct.c_uint64()
    from paper_1811_06127_b200 import _lib

    _lib.check(fn(dix.handle, d_pat.data_ptr(), m, count, d_out.data_ptr(), stream, ct.byref(st), ct.byref(ln)))
    return st.value, ln.value


def random_fetch_peak(lib, device: int) -> float | None:
    """Measured random 32-byte fetches/s over 4 GiB on this GPU (the DRAM request ceiling)."""
    fn = getattr(lib, "fmgx_random_fetch_rate", None)
    if fn is None:
        return None
    fn.argtypes = [ct.c_int, ct.c_uint64, ct.c_uint64, ct.POINTER(ct.c_double)]
    rate = ct.c_double()
    if fn(device, 4 << 30, 1 << 25, ct.byref(rate)) != 0:
        return None
    return rate.value


def fetch_chunks(pairs: np.ndarray, chars_per_chunk: int = 256) -> int:
    """Distinct 128-byte DRAM chunks the W = 2 layout touches per step, summed:
    one chunk holds 4 lines = 256 characters; k-1 and l in the same chunk share it."""
    low, high = pairs[:, 0], pairs[:, 1]
    two = (low >= 0) & ((low // chars_per_chunk) != (high // chars_per_chunk))
    return int(low.size + two.sum())


def occ_layout(lib, dix) -> str:
    """Layout the Occ-step kernel reads for this index: 'lines' (32-byte lines,
    one sector per position) or 'chunks' (128-byte chunks, HBM-resident)."""
    fn = lib.fmgx_occ_layout
    fn.argtypes = [ct.c_void_p, ct.POINTER(ct.c_int)]
    c = ct.c_int()
    from paper_1811_06127_b200 import _lib

    _lib.check(fn(dix.handle, ct.byref(c)))
    return f"chunks{c.value}" if c.value else "lines"


def occ_roofline(lib, dix, pairs: np.ndarray, launch_s: float, device: int, config: str) -> dict:
    """Roofline of one Occ-step launch over `pairs`, for the layout
    the kernel actually reads.  L2-resident index (config 1): the bound is the
    random L2 read rate, measured live on a buffer of the index's size; the
    HBM figure rides along (its frac exceeds 1: index bytes come from L2).
    HBM-resident (config 1-H): HBM bytes at 32-byte sector granularity, plus
    the DRAM random-fetch rate (128-byte fetches) measured live."""
    units = pairs.shape[0]
    layout = occ_layout(lib, dix)
    peak, kind = hbm_peak()
    line_bytes, lines = occ_step_bytes(pairs)
    if layout.startswith("chunks"):
        ns = int(layout[6:])
        alg, sectors, chunks = chunk_step_bytes(pairs, CHUNK_CHARS[ns])
        kernel = f"k_occ_pair_chunk<{ns}>"
    else:
        alg, sectors, chunks = line_bytes, lines, fetch_chunks(pairs)
        kernel = "k_occ_pair"
    achieved = alg / launch_s / 1e9
    hbm = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "traffic": measured_traffic(kernel, config), "peak_kind": kind,
           "kernel": kernel, "layout": layout, "alg_bytes_per_launch": alg,
           "alg_bytes_per_step": round(alg / units, 2), "sectors_per_step": round(sectors / units, 4),
           "random_sector_roofline_steps_per_s": round(peak * 1e9 / (alg / units), 1),
           "line_layout_bytes_per_step": round(line_bytes / units, 2),
           "frac_line_layout_bytes": round(line_bytes / launch_s / 1e9 / peak, 4),
           "note": "algorithmic bytes = 32 B x the distinct sectors the layout must read per step "
                   "(|S(k-1) U S(l)|, exact replay of the pair list) + 8 B in + 32 B out; "
                   "frac_line_layout_bytes: the same time against the 32-byte-line layout's bytes "
                   "(one sector per position, the fewest any layout with in-sector checkpoints reads)"}
    if dix.device_bytes <= (64 << 20) and layout == "lines":
        fn = lib.fmgx_random_fetch_rate
        fn.argtypes = [ct.c_int, ct.c_uint64, ct.c_uint64, ct.POINTER(ct.c_double)]
        rate = ct.c_double()
        if fn(device, max(int(dix.device_bytes), 1 << 20), 1 << 25, ct.byref(rate)) == 0 and rate.value > 0:
            ach = lines / launch_s
            return {"bound": "l2", "achieved": round(ach / 1e9, 2), "peak": round(rate.value / 1e9, 2),
                    "unit": "G random 32-B L2 line reads/s", "frac": round(ach / rate.value, 4),
                    "traffic": measured_traffic(kernel, config), "kernel": kernel, "layout": layout,
                    "peak_kind": "measured live (random 32-B reads over an L2-resident buffer of the index's size)",
                    "lines_per_step": round(lines / units, 4),
                    "note": "the 8.4 MB index is L2-resident, so the Occ step is bound by the SM->L2 random "
                            "request rate, not HBM; the kernel also streams its pairs in and counts out",
                    "hbm": hbm}
        return hbm
    fetch_peak = random_fetch_peak(lib, device)
    if fetch_peak:
        hbm["request_roofline"] = {
            "bound": "dram_random_requests", "achieved": round(chunks / launch_s / 1e9, 2),
            "peak": round(fetch_peak / 1e9, 2),
            "unit": f"G random {32 * int(layout[6:]) if layout.startswith('chunks') else 128}-B fetches/s",
            "frac": round(chunks / launch_s / fetch_peak, 4), "chunks_per_step": round(chunks / units, 4),
            "note": "distinct 128-byte chunks per step (exact replay); peak measured live: random 32-B reads "
                    "over 4 GiB, each fetching 128 B from DRAM; L2 hits let frac exceed 1"}
    return hbm


def hbm_resident_extra(dev, lib, reps: int = 10) -> dict:
    """Config 1-H on the same GPU: the config-1 pair distribution over the 1 Gbp
    config-4 text, whose 500 MB line array cannot live in the 126 MB L2."""
    import torch

    import paper_1811_06127_b200 as fm
    from paper_1811_06127_b200 import _lib, workloads

    wl = workloads.config1h()
    t0 = time.perf_counter()
    idx = fm.build_index(wl.text, builder="gpu", device=dev.index)
    build_s = time.perf_counter() - t0
    dix = idx.device_index(dev.index)
    units = wl.pairs.shape[0]
    kl = np.empty((units, 2), dtype=np.uint32)
    kl[:, 0] = (wl.pairs[:, 0] + 1).astype(np.uint32)
    kl[:, 1] = wl.pairs[:, 1].astype(np.uint32)
    d_kl = torch.from_numpy(kl.view(np.int32)).to(dev)
    d_out = torch.empty((units, 8), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        _lib.check(lib.fmg_occ_pair(dix.handle, d_kl.data_ptr(), units, d_out.data_ptr(), None, stream.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        lib.fmg_occ_pair(dix.handle, d_kl.data_ptr(), units, d_out.data_ptr(), None, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launch_s = e0.elapsed_time(e1) / reps / 1e3
    roof = occ_roofline(lib, dix, wl.pairs, launch_s, dev.index, "config1h")
    idx.release_device()
    return {"workload": "config 1-H: 2^24 config-1 pairs over the 1 Gbp config-4 text (seed 5), "
                        "HBM-resident index (500 MB of lines + the chunk layout the Occ kernel reads)",
            "value": units / launch_s, "unit": "occ_steps/s", "index_build_s_gpu": round(build_s, 2),
            "roofline": roof}


def run_ours(args, rank: int, local: int, world: int) -> None:
    import torch

    import paper_1811_06127_b200 as fm
    from paper_1811_06127_b200 import _lib
    from paper_1811_06127_b200.dist import max_over_ranks

    # one rank per GPU; more ranks than GPUs (a parity run of the N-rank path on
    # a smaller box) share devices round-robin and talk over gloo, since NCCL
    # refuses two ranks on one device — no rank ever waits on another's kernels
    n_dev = torch.cuda.device_count()
    if n_dev == 0:
        raise SystemExit("bench.py: no CUDA device visible — the engine runs only on the GPU (no CPU fallback); "
                         "`--impl reference` times the CPU restatement of the reference")
    oversubscribed = world > n_dev
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    gloo = None
    if world > 1:
        import torch.distributed as dist

        if oversubscribed:
            dist.init_process_group("gloo")
            gloo = None
        else:
            dist.init_process_group("nccl", device_id=dev)
            gloo = dist.new_group(backend="gloo")  # host-side digest gather (off the timed path)
    lib = _lib.load()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    wl = shared_workload(args.config, rank, world, barrier)
    full_wl = wl
    # Configs 3 and 4 define one fixed query set "sharded over 1, 2, 4 and 8
    # GPUs" (strong scaling): rank r keeps its contiguous shard.  The others
    # are weak-scaled (config 1: an independent pair set per rank).
    strong = args.config in ("config3", "config4") and world > 1
    if strong:
        from paper_1811_06127_b200.dist import shard_range

        import copy

        wl = copy.copy(full_wl)
        wl.meta = dict(full_wl.meta)
        if wl.name == "config3":
            per = wl.meta["seeds_per_read"]
            lo, hi = shard_range(wl.meta["reads"], rank, world)
            wl.packed = np.array(full_wl.packed[lo * per:hi * per])
            wl.meta["reads"] = hi - lo
        else:
            lo, hi = shard_range(full_wl.packed.size, rank, world)
            wl.packed = np.array(full_wl.packed[lo:hi])
    # ranks that share a GPU (a parity run on a box with fewer GPUs than ranks) build one after
    # another: the GPU builder wants ~36 bytes per character of device memory (112 GB at 3.1 Gbp)
    share = world > 1 and oversubscribed
    t_build = 0.0
    for turn in range(world if share else 1):
        if not share or turn == rank:
            t_build = time.perf_counter()
            idx = fm.build_index(wl.text)
            t_build = time.perf_counter() - t_build
            dix = idx.device_index(local)
        if share:
            torch.distributed.barrier()
    # a dedicated non-blocking stream: the legacy default stream would
    # serialise against the library's stream-ordered allocations
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    units = unit_count(wl)
    metric, unit = metric_of(args.config)
    extra: dict = {"index_build_s": round(t_build, 2), "index_device_bytes": dix.device_bytes}
    free_b, total_b = torch.cuda.mem_get_info(dev)  # what else holds device memory when the engine sizes its scratch
    extra["gpu_mem_free_after_index"] = int(free_b)
    if wl.max_diff == 1 and wl.pairs is None:
        from paper_1811_06127_b200.search import bidir_min_n

        z1_len = wl.meta["m"] if wl.packed is not None else wl.patterns.shape[1]
        if idx.n >= bidir_min_n() and dix.wants_reverse(units, z1_len, 1):
            # the reversed-text index of the bidirectional z = 1 engines
            t_rev = time.perf_counter()
            dix.ensure_reverse()
            extra["reverse_index_build_s"] = round(time.perf_counter() - t_rev, 2)
            extra["engine"] = ("bidirectional z=1, level-synchronous (spine + chain kernels; L2-resident lines)"
                               if dix.device_bytes <= (64 << 20) else
                               "bidirectional z=1 (case-A / case-B DFS launches + merge)")
        elif idx.n >= bidir_min_n():
            extra["engine"] = ("flat z=1 (k_flat_probe with the neighbourhood presence filter, k_flat_extend, "
                               "k_flat_collect; no reverse index)")
    if wl.pairs is None:  # search configs: the k-mer / prefix interval table, built before timing
        fn = lib.fmgx_prefix_table
        fn.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint64)]
        kk, nb = ct.c_uint32(), ct.c_uint64()
        torch.cuda.synchronize(dev)
        t_lut = time.perf_counter()
        _lib.check(fn(dix.handle, ct.byref(kk), ct.byref(nb)))
        extra["prefix_table"] = {"k": kk.value, "bytes": nb.value,
                                 "build_s": round(time.perf_counter() - t_lut, 4)}
        if wl.name == "config3" or wl.max_diff == 0:  # exact search: its k-mer table (maybe one level deeper)
            fx = lib.fmgx_kmer_table
            fx.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint64)]
            t_lut = time.perf_counter()
            _lib.check(fx(dix.handle, ct.byref(kk), ct.byref(nb)))
            extra["kmer_table"] = {"k": kk.value, "extension_bytes": nb.value,
                                   "build_s": round(time.perf_counter() - t_lut, 4)}

    if wl.name == "config3":
        m = wl.meta["m"]
        n_seeds = wl.packed.size
        d_pat = torch.from_numpy(wl.packed.view(np.int64)).to(dev)
        d_out = torch.empty((n_seeds, 2), dtype=torch.int32, device=dev)
        # z = 1 calls of at most 2^24 seeds, equal-sized (a rank's shard at 8 GPUs, 17.5M seeds,
        # runs as 2 x 8.75M rather than 16.8M + 0.7M)
        call_log2 = int(os.environ.get("FMG_C3_CALL_LOG2", 24))  # A/B: seeds per z = 1 call
        n_chunks = max(1, -(-n_seeds // (1 << call_log2)))
        chunk = -(-n_seeds // n_chunks)
        work_seen = [0, 0, 0]  # inexact Occ steps, lines fetched, kernels launched (library counters, per step)

        def step():
            _lib.check(lib.fmg_exact_packed(dix.handle, d_pat.data_ptr(), m, n_seeds, d_out.data_ptr(), sp))
            for c0 in range(0, n_seeds, chunk):
                h = ct.c_void_p()
                _lib.check(lib.fmg_inexact_packed(dix.handle, d_pat.data_ptr() + 8 * c0, m,
                                                  min(chunk, n_seeds - c0), 1, ct.byref(h), sp))
                st_, ln_, kl_ = ct.c_uint64(), ct.c_uint64(), ct.c_uint64()
                lib.fmg_matches_steps(h, ct.byref(st_))
                lib.fmgx_matches_lines(h, ct.byref(ln_))
                lib.fmgx_matches_launches(h, ct.byref(kl_))
                work_seen[0] += st_.value
                work_seen[1] += ln_.value
                work_seen[2] += kl_.value
                lib.fmg_matches_free(h)

        # the flat engine counts its own launches (k_dbound, then k_flat_probe / _extend / _collect /
        # _advance per chunk of its survivor queue, k_widen_counts, k_gather_matches; CUB scans not
        # counted); the bidirectional split engine: k_dbound, case A + its segment sort, case B + its
        # sort, 2 x k_merge_ab, k_widen_counts, k_gather_matches; + the exact pass
        launches_per_step = 1 + ((n_seeds + chunk - 1) // chunk) * 9
        # the flat engine's three kernels when no reverse index is wanted (HBM-resident index, 19-bp seeds)
        kernel_name = "k_inexact" if "reverse_index_build_s" in extra else "k_flat_probe + k_flat_extend + k_flat_collect"
        h2d_per, d2h_per = n_seeds * 8 * 2, None
        pin_in = torch.from_numpy(wl.packed.view(np.int64)).pin_memory()
        pin_kl = torch.empty((n_seeds, 2), dtype=torch.int32).pin_memory()

        host_res = PinnedResults()
        from concurrent.futures import ThreadPoolExecutor

        copier = ThreadPoolExecutor(max_workers=1)  # result copies of chunk i overlap the search of chunk i+1

        def copy_out(h, cnt):
            try:
                return host_res.copy(lib, h, cnt)
            finally:
                lib.fmg_matches_free(h)

        def e2e_step():
            _lib.check(lib.fmg_exact_packed_host(dix.handle, pin_in.data_ptr(), m, n_seeds, pin_kl.data_ptr()))
            out_bytes = pin_kl.numel() * 4
            pending = []
            for c0 in range(0, n_seeds, chunk):
                h = ct.c_void_p()
                cnt = min(chunk, n_seeds - c0)
                _lib.check(lib.fmg_inexact_packed_host(dix.handle, pin_in.data_ptr() + 8 * c0, m, cnt, 1, ct.byref(h)))
                pending.append(copier.submit(copy_out, h, cnt))
            return out_bytes + sum(f.result() for f in pending)

        alg_bytes = alg_lines = None
        extra["seeds_per_step"] = n_seeds

        def count_work():
            work_seen[0] = work_seen[1] = work_seen[2] = 0
            step()
            torch.cuda.synchronize(dev)
            if work_seen[2]:
                extra["gpu_launches_counted"] = 1 + work_seen[2]
            es, el = exact_work(lib, dix, d_pat, m, n_seeds, d_out, sp)
            return {"exact_steps": es, "exact_lines": el, "inexact_steps": work_seen[0],
                    "inexact_lines": work_seen[1]}
    elif wl.pairs is not None:
        count_work = None
        kl_h = np.empty((units, 2), dtype=np.uint32)
        kl_h[:, 0] = (wl.pairs[:, 0] + 1).astype(np.uint32)
        kl_h[:, 1] = wl.pairs[:, 1].astype(np.uint32)
        d_kl = torch.from_numpy(kl_h.view(np.int32)).to(dev)
        d_out = torch.empty((units, 8), dtype=torch.int32, device=dev)

        d_status = torch.zeros(1, dtype=torch.int32, device=dev)  # per-call input-error word (checked after timing)
        args_ = (dix.handle, d_kl.data_ptr(), units, d_out.data_ptr(), d_status.data_ptr(), sp)  # resolved once

        def step():
            rc = lib.fmg_occ_pair(*args_)
            if rc:
                _lib.check(rc)

        launches_per_step = 1
        kernel_name = "k_occ_pair"
        h2d_per, d2h_per = units * 8, units * 32
        pin_in = torch.from_numpy(kl_h.view(np.int32)).pin_memory()
        pin_out = torch.empty((units, 8), dtype=torch.int32).pin_memory()

        def e2e_step():
            _lib.check(lib.fmg_occ_pair_host(dix.handle, pin_in.data_ptr(), units, pin_out.data_ptr()))
    else:
        m = wl.meta["m"] if wl.packed is not None else wl.patterns.shape[1]
        packed = wl.packed if wl.packed is not None else (fm.pack_patterns_u64(wl.patterns) if m <= 32 else None)
        z = wl.max_diff
        if z == 0 and packed is not None:
            d_pat = torch.from_numpy(packed.view(np.int64)).to(dev)
            d_out = torch.empty((units, 2), dtype=torch.int32, device=dev)

            args_ = (dix.handle, d_pat.data_ptr(), m, units, d_out.data_ptr(), sp)  # resolved once

            def step():
                rc = lib.fmg_exact_packed(*args_)
                if rc:
                    _lib.check(rc)

            launches_per_step = 1
            kernel_name = "k_exact"
            h2d_per, d2h_per = units * 8, units * 8

            def count_work():
                es, el = exact_work(lib, dix, d_pat, m, units, d_out, sp)
                return {"exact_steps": es, "exact_lines": el}
            pin_in = torch.from_numpy(packed.view(np.int64)).pin_memory()
            pin_out = torch.empty((units, 2), dtype=torch.int32).pin_memory()

            def e2e_step():
                _lib.check(lib.fmg_exact_packed_host(dix.handle, pin_in.data_ptr(), m, units, pin_out.data_ptr()))
        else:
            # fixed-length seeds (config 2: 32 bp) travel 2-bit packed, one u64 each
            d_pat = torch.from_numpy(packed.view(np.int64)).to(dev)

            def search():
                h = ct.c_void_p()
                _lib.check(lib.fmg_inexact_packed(dix.handle, d_pat.data_ptr(), m, units, z, ct.byref(h), sp))
                return h

            def step():
                lib.fmg_matches_free(search())

            def count_work():
                h = search()
                st_, ln_ = ct.c_uint64(), ct.c_uint64()
                lib.fmg_matches_steps(h, ct.byref(st_))
                lib.fmgx_matches_lines(h, ct.byref(ln_))
                lib.fmg_matches_free(h)
                return {"inexact_steps": st_.value, "inexact_lines": ln_.value}

            launches_per_step = None  # counted below
            kernel_name = "k_inexact"
            h2d_per, d2h_per = packed.nbytes, None
            pin_pat = torch.from_numpy(packed.view(np.int64)).pin_memory()

            host_res = PinnedResults()

            def e2e_step():
                h = ct.c_void_p()
                _lib.check(lib.fmg_inexact_packed_host(dix.handle, pin_pat.data_ptr(), m, units, z, ct.byref(h)))
                out_bytes = host_res.copy(lib, h, units)
                lib.fmg_matches_free(h)
                return out_bytes
        alg_bytes = alg_lines = None

    # ---- warm-up, then exactly K timed steps bracketed by barrier + sync ----
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    t_ms = ev0.elapsed_time(ev1)
    if wl.pairs is not None and int(d_status.item()):
        raise SystemExit("Occ step reported an input error")
    t_ms = max_over_ranks(t_ms, world, dev)
    ms_step = t_ms / args.steps
    total_units = int(dist_sum(units, world, dev)) if world > 1 else units
    value = total_units * args.steps / (t_ms / 1e3)

    # ---- per-launch kernel time for the roofline (same stream, CUDA events) ----
    roofline = None
    if wl.pairs is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, min(args.steps, 20))
        e0.record(stream)
        for _ in range(reps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        launch_s = e0.elapsed_time(e1) / reps / 1e3
        roofline = occ_roofline(lib, dix, wl.pairs, launch_s, local, args.config)
        kernel_name = roofline["kernel"]

    # ---- search configs: device-counted work (one extra, untimed step) ----
    work = None
    if count_work is not None:
        work = count_work()
        steps_all = sum(v for k_, v in work.items() if k_.endswith("_steps"))
        lines_all = sum(v for k_, v in work.items() if k_.endswith("_lines"))
        step_s = ms_step / 1e3
        peak, peak_kind = hbm_peak()
        alg = 32 * lines_all  # one 32-byte sector per distinct line per executed Occ step
        achieved = alg / step_s / 1e9
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": measured_traffic(kernel_name, args.config),
                    "peak_kind": peak_kind, "kernel": kernel_name if launches_per_step == 1 else
                    f"whole step ({kernel_name} dominant)",
                    "alg_bytes_per_launch": alg, "alg_bytes_per_step": round(alg / max(steps_all, 1), 2),
                    "sectors_per_step": round(lines_all / max(steps_all, 1), 4),
                    "note": "algorithmic bytes = 32 B x lines fetched by the executed Occ steps, counted "
                            "on the device; time = the timed step average"}
        fetch_peak = random_fetch_peak(lib, local) if dix.device_bytes > (256 << 20) else None
        if fetch_peak:
            roofline["request_roofline"] = {
                "bound": "dram_random_requests", "achieved": round(lines_all / step_s / 1e9, 2),
                "peak": round(fetch_peak / 1e9, 2), "unit": "G random line fetches/s",
                "frac": round(lines_all / step_s / fetch_peak, 4),
                "note": "each fetched line counted as one random DRAM request; L2 hits let frac exceed 1"}
        extra["work"] = {**work, "occ_steps_per_unit": round(steps_all / units, 2),
                         "lines_per_unit": round(lines_all / units, 2)}

    # ---- end to end through the C-ABI host entry point ----
    e2e_steps = max(2, min(args.steps, 5))
    e2e_step()
    torch.cuda.synchronize(dev)
    d2h_seen = 0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r = e2e_step()
        if isinstance(r, int):
            d2h_seen = r
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_s = max_over_ranks(e2e_s, world, dev)
    e2e = {"value": total_units / e2e_s, "unit": unit, "h2d_bytes_per_step": h2d_per,
           "d2h_bytes_per_step": d2h_per if d2h_per is not None else d2h_seen}

    # ---- CPU baseline (oracle port) on rank 0 at N=1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc

        ox = orc.OracleIndex(idx)
        th = cpu_threads()
        if wl.name == "config3":
            sample = min(units, 2_000)
            per = wl.meta["seeds_per_read"]
            sp3 = pattern_sample(wl, 0, sample * per)

            def fn():
                orc.exact_batch(ox, sp3, th)
                return orc.inexact_batch(ox, sp3, 1, th)

            if work is not None:  # the reference DFS's own step count per seed, beside ours
                extra["work"]["reference_dfs_steps_per_seed"] = round(fn()[4] / sp3.shape[0], 2)
                extra["work"]["inexact_steps_per_seed"] = round(work["inexact_steps"] / max(1, wl.packed.size), 2)
        elif wl.pairs is not None:
            sample = min(units, 1 << 22)
            fn = lambda: orc.occ_pair_batch(ox, wl.pairs[:sample, 0], wl.pairs[:sample, 1], th)  # noqa: E731
        elif wl.max_diff:
            sample = min(units, 20_000)
            sp_ = pattern_sample(wl, 0, sample)
            fn = lambda: orc.inexact_batch(ox, sp_, wl.max_diff, th)  # noqa: E731
            if work is not None:  # the reference DFS's own step count, beside ours
                extra["work"]["reference_dfs_steps_per_unit"] = round(fn()[4] / sample, 2)
        else:
            sample = min(units, 1 << 20)
            sp_ = pattern_sample(wl, 0, sample)
            fn = lambda: orc.exact_batch(ox, sp_, th)  # noqa: E731
        fn()
        reps, t0 = 0, time.perf_counter()
        while reps < 1 or time.perf_counter() - t0 < 5.0:
            fn()
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": sample / dt, "unit": unit, "cores": th, "kind": "port",
               "sample": f"first {sample} units of the {args.config} workload, {reps} reps; oracle/fm_oracle.c "
                         f"(C restatement of the reference path) on {th} threads of {cpu_model()}"}

    # ---- config 1-H beside config 1 (rank 0, N=1): the HBM-resident regime ----
    if args.config == "config1" and rank == 0 and world == 1 and not args.no_hbm_extra:
        extra["hbm_resident"] = hbm_resident_extra(dev, lib)

    # ---- N > 1: every rank's results, as digests, against rank 0 recomputing
    # that rank's queries on its own GPU (off the timed path) ----
    parity = None
    if world > 1 and not args.no_parity:
        import torch.distributed as dist

        def shard_digest(r: int) -> str:
            if wl.pairs is not None:
                pr = wl.pairs if r == rank else make_workload("config1", r).pairs
                return digest_pairs(fm, idx, pr)
            if strong:
                per = full_wl.meta.get("seeds_per_read", 1)
                total_q = full_wl.meta["reads"] if full_wl.name == "config3" else full_wl.packed.size
                lo_, hi_ = shard_range(total_q, r, world)
                return digest_patterns(lib, dix, full_wl, lo_ * per, hi_ * per)
            return digest_patterns(lib, dix, wl, 0, unit_count(wl))  # weak: every rank runs the same set

        mine = shard_digest(rank)
        got = [None] * world
        dist.all_gather_object(got, mine, group=gloo)
        if rank == 0:
            want = [mine] + [shard_digest(r) for r in range(1, world)]
            parity = {"ok": got == want, "ranks": world,
                      "method": "SHA-256 of each rank's full results (intervals / CSR counts, k, l, diffs / "
                                "Occ counts) gathered to rank 0 and compared with rank 0 recomputing that "
                                "rank's queries with the same engine"}
            if not parity["ok"]:
                print(json.dumps({"error": "multi-rank parity check failed", "got": got, "want": want}),
                      file=sys.stderr, flush=True)

    # ---- launch count: our kernels inside the timed region ----
    if launches_per_step is None:
        # config 2 (level-synchronous bidirectional engine): k_dbound, k_bspine, k_bchain, k_z1_hist_dev,
        # k_widen_counts x2, k_z1_scatter_dev, k_z1_sort_unique, k_z1_write_kl (CUB scans not counted)
        launches_per_step = 9
    if "gpu_launches_counted" in extra:  # the engine counted its own launches for one step
        launches_per_step = extra.pop("gpu_launches_counted")
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "u32", "data": DATA,
            "config": config_of(args.config, world, units),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
            "gpu_launches": launches_per_step * args.steps, **extra,
            **({"parity": parity} if parity is not None else {}),
            **({"oversubscribed": f"{world} ranks on {n_dev} GPU(s): a parity run, not a scaling number"}
               if oversubscribed else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="config1",
                    choices=["config1", "config1h", "config0", "config2", "config3", "config4"])
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hbm-extra", action="store_true", help="skip the config 1-H side measurement")
    ap.add_argument("--no-parity", action="store_true", help="N > 1: skip the gathered-digest parity check")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    rank, local, world = (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
                          int(os.environ.get("WORLD_SIZE", 1)))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, local, world)


if __name__ == "__main__":
    main()
