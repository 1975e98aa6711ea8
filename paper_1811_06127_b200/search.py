"""Backward search, bounded-difference search and position recovery on the GPU.

Mirrors the reference's search module (search.py:1-286) name for name.  The
scalar functions are N = 1 wrappers of the batched entry points:

    exact_search_batch    -> fmg_exact_host / fmg_exact_packed_host (k_exact)
    inexact_search_batch  -> fmg_inexact_host (k_inexact)
    psi_inverse_batch     -> fmg_psi_inverse (k_psi)
    locate_rows           -> fmg_locate_rows_host (k_locate)

Host-side work is limited to argument validation, the pattern gate
(degenerate / empty patterns) and the record bookkeeping of locate_all /
collect_hits (search.py:211-267), done with vectorised numpy.
"""

from __future__ import annotations

import ctypes as ct
import os
from typing import Iterable, NamedTuple

import numpy as np

from . import _lib
from .alphabet import SYMBOLS, encode_array, is_dna, pack_patterns_u64, patterns_to_csr
from .device import require_gpu
from .index import FmIndex, SA_STRIDE
from .kernels import Kernel, resolve_kernel
from .occ import occ_pair_all


class BwmInterval(NamedTuple):
    """Inclusive row range [k, l]; empty when k > l (search.py:14-31)."""

    k: int
    l: int
    degenerate: bool = False

    @property
    def is_empty(self) -> bool:
        return self.k > self.l

    @property
    def width(self) -> int:
        return 0 if self.k > self.l else self.l - self.k + 1


class MatchResult(NamedTuple):
    """One surviving interval of the bounded-difference search (search.py:34-38)."""

    interval: BwmInterval
    diffs_used: int


class Hit(NamedTuple):
    """A located occurrence, mapped to its record (search.py:41-47)."""

    record: str
    offset: int
    global_pos: int
    diffs: int


def init_interval(index: FmIndex, symbol: int) -> BwmInterval:
    """Row range of rotations starting with `symbol`: [c[s]+1, c[s+1]] (search.py:50-57)."""
    if not 0 <= symbol < 4:
        raise ValueError(f"symbol code {symbol} outside [0, 4)")
    return BwmInterval(k=index.c[symbol] + 1, l=index.c[symbol + 1])


def extend_backward(
    index: FmIndex, interval: BwmInterval, symbol: int, kernel: Kernel | str | None = None
) -> BwmInterval:
    """Narrow an interval by one more symbol (search.py:60-71)."""
    if interval.is_empty:
        raise ValueError("cannot extend an empty interval")
    pair = occ_pair_all(index, interval.k - 1, interval.l, kernel)
    c = index.c[symbol]
    return BwmInterval(k=c + pair.at_low[symbol] + 1, l=c + pair.at_high[symbol])


# ---------------------------------------------------------------------------
# exact search
# ---------------------------------------------------------------------------


def exact_search_batch(index: FmIndex, patterns, kernel: Kernel | str | None = None,
                       device: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """exact_search over many patterns in one launch.

    `patterns`: a list of strings, or an (N, m) uint8 array of codes.  Returns
    (kl, degenerate): kl is (N, 2) int64 with the interval exact_search returns
    for each pattern (the first empty interval where the search stopped, or
    (1, 0) for degenerate patterns, search.py:85-86).
    """
    resolve_kernel(kernel)
    lib = _lib.load()
    if isinstance(patterns, np.ndarray) and patterns.ndim == 2 and 1 <= patterns.shape[1] <= 32:
        codes = np.ascontiguousarray(patterns, dtype=np.uint8)
        if codes.size and codes.max() > 3:
            raise ValueError("symbol code outside [0, 4)")
        n = codes.shape[0]
        out = np.empty((n, 2), dtype=np.uint32)
        if n:
            require_gpu()
            dev = index.device_index(device)
            packed = pack_patterns_u64(codes)
            _lib.check(lib.fmg_exact_packed_host(dev.handle, packed.ctypes.data, codes.shape[1], n,
                                                 out.ctypes.data))
        return out.astype(np.int64), np.zeros(n, dtype=bool)
    codes, offsets, degenerate = patterns_to_csr(patterns)
    n = offsets.size - 1
    out = np.empty((n, 2), dtype=np.uint32)
    if n:
        require_gpu()
        dev = index.device_index(device)
        _lib.check(lib.fmg_exact_host(dev.handle, codes.ctypes.data, offsets.ctypes.data, n,
                                      out.ctypes.data))
    kl = out.astype(np.int64)
    kl[degenerate] = (1, 0)
    return kl, degenerate


def exact_search(index: FmIndex, pattern: str, kernel: Kernel | str | None = None) -> BwmInterval:
    """Interval of rows whose rotations start with `pattern` (search.py:74-94)."""
    if not pattern:
        raise ValueError("pattern is empty")
    if not is_dna(pattern):
        return BwmInterval(k=1, l=0, degenerate=True)
    kl, _ = exact_search_batch(index, [pattern], kernel)
    return BwmInterval(k=int(kl[0, 0]), l=int(kl[0, 1]))


# ---------------------------------------------------------------------------
# bounded-difference search
# ---------------------------------------------------------------------------


class MatchSet(NamedTuple):
    """CSR result of inexact_search_batch: pattern i owns rows offsets[i]:offsets[i+1]."""

    offsets: np.ndarray  # (N+1,) uint64
    k: np.ndarray        # (total,) uint32
    l: np.ndarray        # (total,) uint32
    diffs: np.ndarray    # (total,) uint8
    steps: int           # Occ steps executed by the engine

    def results(self, i: int) -> list[MatchResult]:
        a, b = int(self.offsets[i]), int(self.offsets[i + 1])
        return [
            MatchResult(BwmInterval(int(k), int(l)), int(d))
            for k, l, d in zip(self.k[a:b], self.l[a:b], self.diffs[a:b])
        ]

    def __len__(self) -> int:
        return self.offsets.size - 1


BIDIR_MIN_N = 1 << 22


def bidir_min_n() -> int:
    """Index size from which z = 1 batches attach the reversed-text index
    (FMG_BIDIR_MIN_N overrides; the one-directional engines stay exact)."""
    return int(os.environ.get("FMG_BIDIR_MIN_N", BIDIR_MIN_N))


def inexact_search_batch(index: FmIndex, patterns, max_diff: int,
                         kernel: Kernel | str | None = None, device: int | None = None) -> MatchSet:
    """inexact_search over many patterns; results in CSR form (see MatchSet)."""
    if max_diff < 0:
        raise ValueError(f"difference budget {max_diff} is negative")
    if max_diff > 255:  # engine limit (diffs are u8); the reference has none
        raise ValueError(f"difference budget {max_diff} above 255 is not supported")
    resolve_kernel(kernel)
    codes, offsets, degenerate = patterns_to_csr(patterns)
    n = offsets.size - 1
    lib = _lib.load()
    if n == 0:
        return MatchSet(np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.uint32),
                        np.zeros(0, np.uint8), 0)
    require_gpu()
    dev = index.device_index(device)
    if max_diff == 1 and index.n >= bidir_min_n() and n >= 1024:
        max_len = int(np.diff(offsets).max())
        if dev.wants_reverse(n, max_len, max_diff):  # not for the flat engine (kernels_flat.cuh)
            dev.ensure_reverse()  # the bidirectional engines (kernels_bidir.cuh)
    handle = ct.c_void_p()
    _lib.check(lib.fmg_inexact_host(dev.handle, codes.ctypes.data, offsets.ctypes.data, n,
                                    int(max_diff), ct.byref(handle)))
    try:
        total, npat, steps = ct.c_uint64(), ct.c_uint64(), ct.c_uint64()
        _lib.check(lib.fmg_matches_size(handle, ct.byref(total), ct.byref(npat)))
        _lib.check(lib.fmg_matches_steps(handle, ct.byref(steps)))
        row = np.empty(n + 1, dtype=np.uint64)
        k = np.empty(total.value, dtype=np.uint32)
        l = np.empty(total.value, dtype=np.uint32)
        d = np.empty(total.value, dtype=np.uint8)
        _lib.check(lib.fmg_matches_copy(handle, row.ctypes.data, k.ctypes.data, l.ctypes.data,
                                        d.ctypes.data, 1))
    finally:
        lib.fmg_matches_free(handle)
    if degenerate.any():  # search.py:117-118: degenerate patterns yield []
        keep = np.repeat(~degenerate, np.diff(row).astype(np.int64))
        counts = np.diff(row).astype(np.int64)
        counts[degenerate] = 0
        row = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(counts, out=row[1:])
        k, l, d = k[keep], l[keep], d[keep]
    return MatchSet(row, k, l, d, int(steps.value))


def inexact_search(index: FmIndex, pattern: str, max_diff: int,
                   kernel: Kernel | str | None = None) -> list[MatchResult]:
    """All intervals reachable within `max_diff` edits of `pattern` (search.py:97-159)."""
    if max_diff < 0:
        raise ValueError(f"difference budget {max_diff} is negative")
    if not pattern:
        raise ValueError("pattern is empty")
    if not is_dna(pattern):
        return []
    return inexact_search_batch(index, [pattern], max_diff, kernel).results(0)


# ---------------------------------------------------------------------------
# position recovery
# ---------------------------------------------------------------------------


def _check_rows(index: FmIndex, rows: np.ndarray) -> None:
    bad = (rows < 0) | (rows > index.n)
    if bad.any():
        i = int(rows[np.flatnonzero(bad)[0]])
        raise ValueError(f"row {i} outside [0, {index.n}]")


def psi_inverse_batch(index: FmIndex, rows, device: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(symbol, predecessor row) per row; symbol 255 / row -1 at the sentinel row."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    _check_rows(index, rows)
    n = rows.size
    sym = np.empty(n, dtype=np.uint8)
    prev = np.empty(n, dtype=np.uint32)
    if n:
        require_gpu()
        import torch

        dev = index.device_index(device)
        d_rows = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).to(f"cuda:{dev.device}")
        d_sym = torch.empty(n, dtype=torch.uint8, device=d_rows.device)
        d_prev = torch.empty(n, dtype=torch.int32, device=d_rows.device)
        d_status = torch.zeros(1, dtype=torch.int32, device=d_rows.device)
        stream = torch.cuda.current_stream(dev.device)
        _lib.check(_lib.load().fmg_psi_inverse(dev.handle, d_rows.data_ptr(), n, d_sym.data_ptr(),
                                               d_prev.data_ptr(), d_status.data_ptr(), stream.cuda_stream))
        if int(d_status.item()):  # rows were range-checked above: only a corrupt index gets here
            raise RuntimeError("fmgpu: psi_inverse reported an input error on validated rows")
        sym[:] = d_sym.cpu().numpy()
        prev[:] = d_prev.cpu().numpy().view(np.uint32)
    return sym, np.where(sym == 255, -1, prev.astype(np.int64))


def psi_inverse_fused(index: FmIndex, i: int, kernel: Kernel | str | None = None) -> tuple[int, int] | None:
    """(symbol at row i, predecessor row), None at the sentinel (search.py:172-186)."""
    if not 0 <= i <= index.n:
        raise ValueError(f"row {i} outside [0, {index.n}]")
    resolve_kernel(kernel)
    sym, prev = psi_inverse_batch(index, [i])
    return None if sym[0] == 255 else (int(sym[0]), int(prev[0]))


def psi_inverse(index: FmIndex, i: int, kernel: Kernel | str | None = None) -> int | None:
    """Row of the suffix one position earlier in the text (search.py:162-169)."""
    stepped = psi_inverse_fused(index, i, kernel)
    return None if stepped is None else stepped[1]


def locate_rows(index: FmIndex, rows, device: int | None = None) -> np.ndarray:
    """Text position of every row (search.py:189-208), one GPU launch."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    _check_rows(index, rows)
    out = np.empty(rows.size, dtype=np.uint32)
    if rows.size:
        require_gpu()
        dev = index.device_index(device)
        dev.ensure_samples()
        r32 = rows.astype(np.uint32)
        _lib.check(_lib.load().fmg_locate_rows_host(dev.handle, r32.ctypes.data, r32.size,
                                                    out.ctypes.data))
    return out.astype(np.int64)


def locate_row(index: FmIndex, i: int, kernel: Kernel | str | None = None) -> int:
    """Text position of row i (search.py:189-208)."""
    resolve_kernel(kernel)
    return int(locate_rows(index, [i])[0])


def _hits_from_positions(index: FmIndex, pos: np.ndarray, diffs: np.ndarray,
                         pattern_len: int) -> list[Hit]:
    """search.py:226-242: drop pos >= n and spans forced across a record boundary."""
    starts = np.array([r.start for r in index.records], dtype=np.int64)
    lengths = np.array([r.length for r in index.records], dtype=np.int64)
    keep = pos < index.n
    pos, diffs = pos[keep], diffs[keep]
    which = np.searchsorted(starts, pos, side="right") - 1
    offset = pos - starts[which]
    min_span = np.maximum(pattern_len - diffs, 0)
    ok = offset + min_span <= lengths[which]
    pos, diffs, which, offset = pos[ok], diffs[ok], which[ok], offset[ok]
    order = np.argsort(pos, kind="stable")
    names = [r.name for r in index.records]
    return [
        Hit(record=names[int(which[j])], offset=int(offset[j]), global_pos=int(pos[j]),
            diffs=int(diffs[j]))
        for j in order
    ]


def locate_all(index: FmIndex, interval: BwmInterval, diffs: int, pattern_len: int,
               kernel: Kernel | str | None = None) -> list[Hit]:
    """Map every row of an interval to a record-relative hit (search.py:211-242)."""
    if interval.is_empty:
        return []
    resolve_kernel(kernel)
    pos = locate_rows(index, np.arange(interval.k, interval.l + 1, dtype=np.int64))
    return _hits_from_positions(index, pos, np.full(pos.size, diffs, dtype=np.int64), pattern_len)


def collect_hits(index: FmIndex, matches: Iterable[MatchResult], pattern_len: int,
                 kernel: Kernel | str | None = None, max_hits: int | None = None) -> tuple[list[Hit], bool]:
    """Merge hits of several intervals, fewest diffs per position (search.py:245-267)."""
    resolve_kernel(kernel)
    ms = sorted(matches, key=lambda m: m.diffs_used)
    rows, dif = [], []
    for m in ms:
        if not m.interval.is_empty:
            rows.append(np.arange(m.interval.k, m.interval.l + 1, dtype=np.int64))
            dif.append(np.full(m.interval.width, m.diffs_used, dtype=np.int64))
    if rows:
        rows_a, dif_a = np.concatenate(rows), np.concatenate(dif)
        pos = locate_rows(index, rows_a)
        # per-interval filtering first (locate_all semantics), then min-diff merge
        starts = np.array([r.start for r in index.records], dtype=np.int64)
        lengths = np.array([r.length for r in index.records], dtype=np.int64)
        keep = pos < index.n
        pos, dif_a = pos[keep], dif_a[keep]
        which = np.searchsorted(starts, pos, side="right") - 1
        offset = pos - starts[which]
        ok = offset + np.maximum(pattern_len - dif_a, 0) <= lengths[which]
        pos, dif_a, which, offset = pos[ok], dif_a[ok], which[ok], offset[ok]
        # smallest diffs per position; ties keep the first (lowest-diff interval order)
        order = np.lexsort((dif_a, pos))
        pos, dif_a, which, offset = pos[order], dif_a[order], which[order], offset[order]
        first = np.ones(pos.size, dtype=bool)
        first[1:] = pos[1:] != pos[:-1]
        pos, dif_a, which, offset = pos[first], dif_a[first], which[first], offset[first]
        names = [r.name for r in index.records]
        hits = [Hit(names[int(w)], int(o), int(p), int(d)) for w, o, p, d in zip(which, offset, pos, dif_a)]
    else:
        hits = []
    truncated = max_hits is not None and len(hits) > max_hits
    if truncated:
        hits = hits[:max_hits]
    return hits, truncated


def reconstruct_codes(index: FmIndex, device: int | None = None) -> np.ndarray:
    """The n text codes the index was built from, recovered on the GPU.

    Parallel form of reconstruct_reference (search.py:270-286): every sampled
    row starts a predecessor walk of ~32 steps (k_reconstruct), together
    covering the whole cycle from row 0 to the sentinel row.
    """
    require_gpu()
    dev = index.device_index(device)
    dev.ensure_samples()
    out = np.empty(index.n, dtype=np.uint8)
    _lib.check(_lib.load().fmg_reconstruct_text_host(dev.handle, out.ctypes.data))
    return out


def reconstruct_reference(index: FmIndex, kernel: Kernel | str | None = None) -> str:
    """Rebuild the reference text (search.py:270-286) on the GPU (reconstruct_codes)."""
    resolve_kernel(kernel)
    lut = np.frombuffer(SYMBOLS.encode(), dtype=np.uint8)
    return lut[reconstruct_codes(index)].tobytes().decode("ascii")


def collect_hits_batch(index: FmIndex, pid: np.ndarray, k: np.ndarray, l: np.ndarray, diffs: np.ndarray,
                       pattern_len: np.ndarray, max_hits: int | None = None):
    """collect_hits (search.py:245-267) for many patterns with ONE locate launch.

    Intervals are given flat: pattern id, k, l, diffs per matched interval
    (empty intervals allowed and ignored); pattern_len[p] is the length of
    pattern p.  Returns (hit_pid, positions, diffs, record index, offset)
    sorted by (pattern, position), the fewest diffs per position, and the
    per-pattern `truncated` flags of max_hits.
    """
    pid = np.asarray(pid, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    l = np.asarray(l, dtype=np.int64)
    diffs = np.asarray(diffs, dtype=np.int64)
    n_pat = int(np.asarray(pattern_len).size)
    live = l >= k
    pid, k, l, diffs = pid[live], k[live], l[live], diffs[live]
    width = l - k + 1
    total = int(width.sum())
    if total == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z, z, z, z, np.zeros(n_pat, dtype=bool)
    owner = np.repeat(np.arange(width.size), width)
    starts = np.zeros(width.size, dtype=np.int64)
    np.cumsum(width[:-1], out=starts[1:])
    rows = k[owner] + (np.arange(total, dtype=np.int64) - starts[owner])
    pos = locate_rows(index, rows)
    hp, hd = pid[owner], diffs[owner]
    # locate_all filters (search.py:226-238), per interval's own diffs
    rec_start = np.array([r.start for r in index.records], dtype=np.int64)
    rec_len = np.array([r.length for r in index.records], dtype=np.int64)
    keep = pos < index.n
    pos, hp, hd = pos[keep], hp[keep], hd[keep]
    which = np.searchsorted(rec_start, pos, side="right") - 1
    offset = pos - rec_start[which]
    plen = np.asarray(pattern_len, dtype=np.int64)[hp]
    ok = offset + np.maximum(plen - hd, 0) <= rec_len[which]
    pos, hp, hd, which, offset = pos[ok], hp[ok], hd[ok], which[ok], offset[ok]
    # fewest diffs per (pattern, position), sorted by (pattern, position)
    order = np.lexsort((hd, pos, hp))
    pos, hp, hd, which, offset = pos[order], hp[order], hd[order], which[order], offset[order]
    first = np.ones(pos.size, dtype=bool)
    first[1:] = (pos[1:] != pos[:-1]) | (hp[1:] != hp[:-1])
    pos, hp, hd, which, offset = pos[first], hp[first], hd[first], which[first], offset[first]
    truncated = np.zeros(n_pat, dtype=bool)
    if max_hits is not None:
        group_start = np.zeros(hp.size, dtype=np.int64)
        new = np.ones(hp.size, dtype=bool)
        new[1:] = hp[1:] != hp[:-1]
        idx_new = np.flatnonzero(new)
        group_start[idx_new] = idx_new
        group_start = np.maximum.accumulate(group_start)
        rank = np.arange(hp.size) - group_start
        over = rank >= max_hits
        truncated[np.unique(hp[over])] = True
        keep = ~over
        pos, hp, hd, which, offset = pos[keep], hp[keep], hd[keep], which[keep], offset[keep]
    return hp, pos, hd, which, offset, truncated
