"""ctypes wrapper of the CPU oracle (fm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker and the CPU
baseline; the product package never imports it.  Each function restates the
reference function cited beside it (see fm_oracle.c for line references)
over the index's .fmi bucket records.
"""

from __future__ import annotations

import ctypes as ct
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"


class _Index(ct.Structure):
    _fields_ = [
        ("rec", ct.c_void_p),
        ("nb", ct.c_uint64),
        ("n", ct.c_uint64),
        ("sentinel_row", ct.c_uint64),
        ("c", ct.c_uint64 * 5),
        ("samples", ct.c_void_p),
    ]


def build(force: bool = False) -> Path:
    newest = max((HERE / f).stat().st_mtime for f in ("fm_oracle.c", "fm_build.c", "Makefile"))
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return LIB


_lib = None


def load():
    global _lib
    if _lib is None:
        build()
        lib = ct.CDLL(str(LIB))
        vp, u64 = ct.c_void_p, ct.c_uint64
        lib.fmo_occ_pair_batch.argtypes = [vp, vp, vp, u64, vp, ct.c_int]
        lib.fmo_exact_batch.argtypes = [vp, vp, vp, u64, vp, ct.c_int]
        lib.fmo_locate_batch.argtypes = [vp, vp, u64, vp, ct.c_int]
        lib.fmo_inexact_batch.argtypes = [vp, vp, vp, u64, ct.c_int64, ct.c_int]
        lib.fmo_inexact_batch.restype = vp
        lib.fmo_matches_total.argtypes = [vp]
        lib.fmo_matches_total.restype = u64
        lib.fmo_matches_steps.argtypes = [vp]
        lib.fmo_matches_steps.restype = u64
        lib.fmo_matches_fetch.argtypes = [vp, vp, vp, vp, vp]
        lib.fmo_matches_free.argtypes = [vp]
        lib.fmo_psi.argtypes = [vp, ct.c_int64, ct.POINTER(ct.c_int)]
        lib.fmo_psi.restype = ct.c_int64
        lib.fmo_build_sa.argtypes = [vp, u64, vp, ct.c_int]
        lib.fmo_build_records.argtypes = [vp, u64, vp, vp, vp, vp, vp]
        _lib = lib
    return _lib


def threads_default() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class BuiltIndex:
    """An index built by the oracle's own restatement of the reference build
    (fm_build.c: build_suffix_array, bwt_from_sa, build_index), with the
    attributes OracleIndex reads.  Never touches the product library."""

    def __init__(self, codes, threads: int | None = None, keep_sa: bool = False):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        n = codes.size
        if n == 0:
            raise ValueError("reference is empty")
        lib = load()
        sa = np.empty(n + 1, dtype=np.uint32)
        if lib.fmo_build_sa(codes.ctypes.data, n, sa.ctypes.data, threads or threads_default()):
            raise MemoryError("oracle suffix sort failed")
        nb = n // 128 + 1
        self.bucket_records = np.empty((nb, 64), dtype=np.uint8)
        self.sa_samples = np.empty(n // 32 + 1, dtype=np.uint64)
        c = np.zeros(5, dtype=np.uint64)
        srow = ct.c_uint64()
        if lib.fmo_build_records(codes.ctypes.data, n, sa.ctypes.data, self.bucket_records.ctypes.data,
                                 self.sa_samples.ctypes.data, c.ctypes.data, ct.byref(srow)):
            raise RuntimeError("oracle build: no suffix at position 0")
        self.n = n
        self.c = tuple(int(x) for x in c)
        self.sentinel_row = int(srow.value)
        self.sa = sa if keep_sa else None


class OracleIndex:
    """Oracle view of an index: bucket records + n, c, sentinel_row, samples."""

    def __init__(self, index):
        self._keep = (np.ascontiguousarray(index.bucket_records),
                      np.ascontiguousarray(index.sa_samples, dtype=np.uint64))
        s = _Index()
        s.rec = self._keep[0].ctypes.data
        s.nb = self._keep[0].shape[0]
        s.n = index.n
        s.sentinel_row = index.sentinel_row
        for i in range(5):
            s.c[i] = index.c[i]
        s.samples = self._keep[1].ctypes.data
        self.struct = s
        self.n = index.n

    @property
    def ref(self):
        return ct.byref(self.struct)


def occ_pair_batch(ox: OracleIndex, low, high, threads: int | None = None) -> np.ndarray:
    """occ_pair_all(index, low[i], high[i]) for every i -> (N, 8) uint32 (occ.py:59-96)."""
    low = np.ascontiguousarray(low, dtype=np.int64)
    high = np.ascontiguousarray(high, dtype=np.int64)
    out = np.empty((low.size, 8), dtype=np.uint32)
    rc = load().fmo_occ_pair_batch(ox.ref, low.ctypes.data, high.ctypes.data, low.size, out.ctypes.data,
                                   threads or threads_default())
    if rc:
        raise ValueError("oracle: position out of range or pair out of order")
    return out


def _csr(patterns):
    if isinstance(patterns, np.ndarray):
        codes = np.ascontiguousarray(patterns, dtype=np.uint8)
        n, m = codes.shape
        return codes.reshape(-1), np.arange(0, (n + 1) * m, m, dtype=np.uint64)
    lut = {ch: i for i, ch in enumerate("ACGT")}
    lut.update({ch.lower(): i for i, ch in enumerate("ACGT")})
    codes = np.array([lut[ch] for p in patterns for ch in p], dtype=np.uint8)
    offs = np.zeros(len(patterns) + 1, dtype=np.uint64)
    np.cumsum([len(p) for p in patterns], out=offs[1:])
    return codes, offs


def exact_batch(ox: OracleIndex, patterns, threads: int | None = None) -> np.ndarray:
    """exact_search per pattern -> (N, 2) int64 (k, l) (search.py:74-94)."""
    codes, offs = _csr(patterns)
    n = offs.size - 1
    out = np.empty((n, 2), dtype=np.int64)
    load().fmo_exact_batch(ox.ref, codes.ctypes.data, offs.ctypes.data, n, out.ctypes.data,
                           threads or threads_default())
    return out


def inexact_batch(ox: OracleIndex, patterns, max_diff: int, threads: int | None = None):
    """inexact_search per pattern -> (row_offsets, k, l, diffs, steps) (search.py:97-159)."""
    codes, offs = _csr(patterns)
    n = offs.size - 1
    lib = load()
    h = lib.fmo_inexact_batch(ox.ref, codes.ctypes.data, offs.ctypes.data, n, int(max_diff),
                              threads or threads_default())
    if not h:
        raise MemoryError("oracle inexact batch failed")
    try:
        total = lib.fmo_matches_total(h)
        row = np.empty(n + 1, dtype=np.uint64)
        k = np.empty(total, dtype=np.int64)
        l = np.empty(total, dtype=np.int64)
        d = np.empty(total, dtype=np.uint8)
        lib.fmo_matches_fetch(h, row.ctypes.data, k.ctypes.data, l.ctypes.data, d.ctypes.data)
        steps = lib.fmo_matches_steps(h)
    finally:
        lib.fmo_matches_free(h)
    return row, k, l, d, int(steps)


def locate_batch(ox: OracleIndex, rows, threads: int | None = None) -> np.ndarray:
    """locate_row per row (search.py:189-208)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(rows.size, dtype=np.int64)
    load().fmo_locate_batch(ox.ref, rows.ctypes.data, rows.size, out.ctypes.data,
                            threads or threads_default())
    return out


def psi(ox: OracleIndex, i: int):
    """psi_inverse_fused (search.py:172-186): (sym, row) or None."""
    sym = ct.c_int()
    r = load().fmo_psi(ox.ref, int(i), ct.byref(sym))
    if r == -2:
        raise ValueError(f"row {i} outside [0, {ox.n}]")
    return None if r == -1 else (sym.value, int(r))


def collect_hits(ox: OracleIndex, pid, k, l, diffs, pattern_len, record_starts=(0,), record_lens=None,
                 threads: int | None = None):
    """collect_hits over many patterns (search.py:211-267, locate_all + collect_hits):
    every row of every non-empty interval located with the oracle's locate_row;
    hits at positions >= n dropped; a hit is kept only if offset + max(m - d, 0)
    fits its record; the fewest diffs per (pattern, position); sorted by
    (pattern, position).  Returns (pid, pos, diffs) int64 arrays."""
    pid = np.asarray(pid, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    l = np.asarray(l, dtype=np.int64)
    diffs = np.asarray(diffs, dtype=np.int64)
    live = l >= k
    pid, k, l, diffs = pid[live], k[live], l[live], diffs[live]
    width = l - k + 1
    owner = np.repeat(np.arange(width.size), width)
    first = np.zeros(width.size, dtype=np.int64)
    np.cumsum(width[:-1], out=first[1:])
    rows = k[owner] + (np.arange(int(width.sum()), dtype=np.int64) - first[owner])
    pos = locate_batch(ox, rows, threads)
    hp, hd = pid[owner], diffs[owner]
    keep = pos < ox.n
    pos, hp, hd = pos[keep], hp[keep], hd[keep]
    starts = np.asarray(record_starts, dtype=np.int64)
    lens = np.asarray(record_lens if record_lens is not None else [ox.n], dtype=np.int64)
    which = np.searchsorted(starts, pos, side="right") - 1
    plen = np.asarray(pattern_len, dtype=np.int64)[hp]
    ok = pos - starts[which] + np.maximum(plen - hd, 0) <= lens[which]
    pos, hp, hd = pos[ok], hp[ok], hd[ok]
    order = np.lexsort((hd, pos, hp))
    pos, hp, hd = pos[order], hp[order], hd[order]
    uniq = np.ones(pos.size, dtype=bool)
    uniq[1:] = (pos[1:] != pos[:-1]) | (hp[1:] != hp[:-1])
    return hp[uniq], pos[uniq], hd[uniq]
