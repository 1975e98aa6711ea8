"""CPU restatement of the reference's bucket-level kernels (numpy, vectorised).

TEST INFRASTRUCTURE ONLY (see oracle.py).  Restates, over N buckets at once:

  count_bucket_scalar   kernels.py:137-144   per-field unpack and compare
  mask_bucket           kernels.py:125-134   fields >= prefix_len zeroed
  count_bucket_nibble   kernels.py:161-211   the three-phase half-byte
                                             pipeline, with its trace
  NibbleTables          kernels.py:53-77

Pinned against the reference's own outputs (tests/golden/buckets.npz,
written by tests/golden/make_golden.py from fmpm.kernels).
"""

from __future__ import annotations

import numpy as np

_SHIFTS = np.arange(4, dtype=np.uint8) * 2


def fields(blocks: np.ndarray) -> np.ndarray:
    """(N, 128) symbol codes of (N, 32) packed buckets (field j in bits 2j of byte j/4)."""
    b = np.asarray(blocks, dtype=np.uint8).reshape(-1, 32)
    return ((b[:, :, None] >> _SHIFTS[None, None, :]) & 3).reshape(-1, 128)


def count_scalar(blocks, prefix_lens, symbols) -> np.ndarray:
    """count_bucket_scalar per bucket: occurrences of symbols[i] in fields [0, prefix_lens[i])."""
    f = fields(blocks)
    pl = np.asarray(prefix_lens, dtype=np.int64).reshape(-1, 1)
    sy = np.asarray(symbols, dtype=np.int64).reshape(-1, 1)
    live = np.arange(128)[None, :] < pl
    return ((f == sy) & live).sum(axis=1)


def all4_scalar(blocks, prefix_lens) -> np.ndarray:
    """(N, 4) counts of A, C, G, T in fields [0, prefix_lens[i])."""
    return np.stack([count_scalar(blocks, prefix_lens, np.full(len(prefix_lens), s)) for s in range(4)], axis=1)


def mask(blocks, prefix_lens) -> np.ndarray:
    """mask_bucket per bucket."""
    b = np.asarray(blocks, dtype=np.uint8).reshape(-1, 32)
    pl = np.asarray(prefix_lens, dtype=np.int64)
    f = fields(b)
    f = np.where(np.arange(128)[None, :] < pl[:, None], f, 0).astype(np.uint8)
    g = f.reshape(-1, 32, 4)
    return (g[:, :, 0] | (g[:, :, 1] << 2) | (g[:, :, 2] << 4) | (g[:, :, 3] << 6)).astype(np.uint8)


def tables() -> tuple[np.ndarray, np.ndarray]:
    """NibbleTables.build(): (lo, hi) 16-entry uint8 tables."""
    v = np.arange(16)
    hi = ((1 << ((v & 3) << 1)) + (1 << (((v >> 2) & 3) << 1))).astype(np.uint8)
    return (~hi).astype(np.uint8), hi


def nibble_trace(blocks, prefix_lens, symbols) -> np.ndarray:
    """(N, 15) uint64 in the layout of fmg_bucket_nibble_trace_host:
    masked words[4], lookup lo words[4], lookup hi words[4], group SADs
    (16 bits each), sad_total | raw_count << 32, count."""
    lo_t, hi_t = tables()
    m = mask(blocks, prefix_lens)
    pl = np.asarray(prefix_lens, dtype=np.int64)
    sy = np.asarray(symbols, dtype=np.int64)
    n = m.shape[0]
    out = np.zeros((n, 15), dtype=np.uint64)
    lo_b = lo_t[m & 0x0F]                       # phase 1: lookups per byte
    hi_b = hi_t[m >> 4]
    out[:, 0:4] = m.view("<u8")
    out[:, 4:8] = lo_b.view("<u8")
    out[:, 8:12] = hi_b.view("<u8")
    sh = (sy * 2).astype(np.uint64)[:, None]
    slo = (lo_b.view("<u8") >> sh) | np.uint64(0xFCFCFCFCFCFCFCFC)   # phase 2
    shi = (hi_b.view("<u8") >> sh) & np.uint64(0x0303030303030303)
    diff = np.abs(slo.view(np.uint8).astype(np.int32) - shi.view(np.uint8).astype(np.int32))  # phase 3
    sads = diff.reshape(n, 4, 8).sum(axis=2).astype(np.uint64)
    total = sads.sum(axis=1)
    raw = np.uint64(8160) - total
    count = np.where(sy == 0, raw.astype(np.int64) - (128 - pl), raw.astype(np.int64))
    out[:, 12] = sads[:, 0] | (sads[:, 1] << np.uint64(16)) | (sads[:, 2] << np.uint64(32)) | (sads[:, 3] << np.uint64(48))
    out[:, 13] = total | (raw << np.uint64(32))
    out[:, 14] = count.astype(np.uint64)
    return out
