"""Bucket-level counting kernels and kernel selection (kernels.py:1-358).

The reference counts symbols inside one 128-character packed bucket through a
plugin registry: Kernel {scalar, bytelut, nibble, simd, auto}, chosen by
argument > FMPM_KERNEL > auto (kernels.py:295-350).  Here every count runs on
the GPU, through two batched sm_100a kernels (csrc/kernels_bucket.cuh):

* popcount (serves ``scalar``, ``bytelut``, ``auto``): masked popcount over the
  bucket's four words, the arithmetic of the Occ-step kernels;
* nibble (serves ``nibble``, ``simd``): the paper's three-phase half-byte
  pipeline (kernels.py:161-211) on GPU byte instructions — 16-entry table
  lookups by byte permute, shift / fill / mask extraction, 4-byte SAD
  aggregation — with the reference's intermediate values available through
  ``KernelTrace``.

Both are bit-exact with the reference on every bucket and prefix length
(tests/test_gpu_buckets.py).  The index-level functions (occ*, searches)
accept ``kernel=`` and validate it the same way; they always use the Occ-step
kernels, whose counting is the popcount method.  The scalar functions here
are N=1 wrappers of the batched forms ``count_bucket_batch``,
``count_bucket_all4_batch`` and ``mask_bucket_batch``.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, NamedTuple

import numpy as np

from . import _lib

BUCKET_CHARS = 128
BUCKET_BYTES = 32
ENV_KERNEL = "FMPM_KERNEL"


class OccCounts(NamedTuple):
    """Per-symbol counts in A, C, G, T order (kernels.py:44-50)."""

    a: int
    c: int
    g: int
    t: int


class NibbleTables(NamedTuple):
    """16-entry tables indexed by a half-byte (kernels.py:53-77).

    hi[v] packs the count of each symbol s among the two fields of v into
    bits 2s..2s+1; lo[v] is its complement.  The GPU nibble kernel holds the
    same tables as compile-time constants (kernels_bucket.cuh: nibble_lut).
    """

    lo: bytes
    hi: bytes

    @staticmethod
    def build() -> "NibbleTables":
        v = np.arange(16)
        hi = (1 << ((v & 3) << 1)) + (1 << (((v >> 2) & 3) << 1))
        return NibbleTables(lo=bytes(((~hi) & 0xFF).astype(np.uint8)), hi=bytes(hi.astype(np.uint8)))


TABLES = NibbleTables.build()


@dataclass
class KernelTrace:
    """Intermediate values of one nibble-kernel call (kernels.py:101-115),
    read back from the GPU pipeline; filled only when passed explicitly."""

    masked_words: list[int] = field(default_factory=list)
    lookup_lo_words: list[int] = field(default_factory=list)
    lookup_hi_words: list[int] = field(default_factory=list)
    group_sads: list[int] = field(default_factory=list)
    sad_total: int = 0
    raw_count: int = 0
    count: int = 0


class Kernel(str, Enum):
    SCALAR = "scalar"
    BYTELUT = "bytelut"
    NIBBLE = "nibble"
    SIMD = "simd"
    AUTO = "auto"
    GPU = "gpu"


# Kernels selectable by name; AUTO resolves before dispatch (kernels.py:307).
CONCRETE_KERNELS = (Kernel.SCALAR, Kernel.BYTELUT, Kernel.NIBBLE, Kernel.SIMD)

# GPU method behind each concrete name: 0 = masked popcount, 1 = nibble pipeline.
_METHOD = {Kernel.SCALAR: 0, Kernel.BYTELUT: 0, Kernel.GPU: 0, Kernel.NIBBLE: 1, Kernel.SIMD: 1}


def resolve_kernel(kernel: Kernel | str | None = None) -> Kernel:
    """Normalise a kernel selection the way the reference does (kernels.py:323-342).

    None consults FMPM_KERNEL, falling back to auto; auto resolves to
    bytelut; an unknown name raises ValueError.  ``gpu`` (this package's own
    name for its popcount method) is accepted too.
    """
    if type(kernel) is Kernel:
        return Kernel.BYTELUT if kernel is Kernel.AUTO else kernel
    if kernel is None:
        kernel = os.environ.get(ENV_KERNEL) or Kernel.AUTO
    try:
        kernel = Kernel(kernel)
    except ValueError:
        names = ", ".join(k.value for k in Kernel)
        raise ValueError(f"unknown kernel {kernel!r}; expected one of: {names}") from None
    return Kernel.BYTELUT if kernel is Kernel.AUTO else kernel


def _device() -> int:
    from .device import current_device, require_gpu

    require_gpu()
    return current_device()


def _check_bucket(block: bytes, prefix_len: int) -> None:
    """kernels.py:118-122."""
    if len(block) != BUCKET_BYTES:
        raise ValueError(f"bucket block must be {BUCKET_BYTES} bytes, got {len(block)}")
    if not 0 <= prefix_len <= BUCKET_CHARS:
        raise ValueError(f"prefix_len {prefix_len} outside [0, {BUCKET_CHARS}]")


def _batch_args(blocks, prefix_lens, symbols=None):
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.uint8).reshape(-1, BUCKET_BYTES))
    pl = np.asarray(prefix_lens, dtype=np.int64).reshape(-1)
    if pl.size != b.shape[0]:
        raise ValueError("one prefix_len per bucket block is required")
    if pl.size and (pl.min() < 0 or pl.max() > BUCKET_CHARS):
        bad = int(pl[(pl < 0) | (pl > BUCKET_CHARS)][0])
        raise ValueError(f"prefix_len {bad} outside [0, {BUCKET_CHARS}]")
    pl = np.ascontiguousarray(pl, dtype=np.uint32)
    sy = None
    if symbols is not None:
        s = np.broadcast_to(np.asarray(symbols, dtype=np.int64), pl.shape)
        if s.size and (s.min() < 0 or s.max() > 3):
            raise ValueError(f"symbol code {int(s[(s < 0) | (s > 3)][0])} outside [0, 4)")
        sy = np.ascontiguousarray(s, dtype=np.uint8)
    return b, pl, sy


def count_bucket_batch(blocks, prefix_lens, symbols, kernel: Kernel | str | None = None) -> np.ndarray:
    """Count of symbols[i] among the first prefix_lens[i] fields of blocks[i]
    for N buckets in one launch -> (N,) uint32."""
    method = _METHOD[resolve_kernel(kernel)]
    b, pl, sy = _batch_args(blocks, prefix_lens, symbols)
    out = np.zeros(pl.size, dtype=np.uint32)
    if pl.size:
        _lib.check(_lib.load().fmg_bucket_count_host(_device(), b.ctypes.data, pl.ctypes.data, sy.ctypes.data,
                                                     pl.size, method, out.ctypes.data))
    return out


def count_bucket_all4_batch(blocks, prefix_lens, kernel: Kernel | str | None = None) -> np.ndarray:
    """All four counts per bucket prefix for N buckets in one launch -> (N, 4) uint32."""
    method = _METHOD[resolve_kernel(kernel)]
    b, pl, _ = _batch_args(blocks, prefix_lens)
    out = np.zeros((pl.size, 4), dtype=np.uint32)
    if pl.size:
        _lib.check(_lib.load().fmg_bucket_count_host(_device(), b.ctypes.data, pl.ctypes.data, None, pl.size,
                                                     method, out.ctypes.data))
    return out


def mask_bucket_batch(blocks, prefix_lens) -> np.ndarray:
    """mask_bucket for N buckets in one launch -> (N, 32) uint8."""
    b, pl, _ = _batch_args(blocks, prefix_lens)
    out = np.zeros_like(b)
    if pl.size:
        _lib.check(_lib.load().fmg_bucket_mask_host(_device(), b.ctypes.data, pl.ctypes.data, pl.size,
                                                    out.ctypes.data))
    return out


def nibble_trace_batch(blocks, prefix_lens, symbols) -> np.ndarray:
    """(N, 15) uint64 traces of the GPU nibble pipeline (layout: include/fmgpu.h)."""
    b, pl, sy = _batch_args(blocks, prefix_lens, symbols)
    out = np.zeros((pl.size, 15), dtype=np.uint64)
    if pl.size:
        _lib.check(_lib.load().fmg_bucket_nibble_trace_host(_device(), b.ctypes.data, pl.ctypes.data,
                                                            sy.ctypes.data, pl.size, out.ctypes.data))
    return out


def mask_bucket(block: bytes, prefix_len: int) -> bytes:
    """Zero every field at positions >= prefix_len (kernels.py:125-134)."""
    if prefix_len >= BUCKET_CHARS:
        return bytes(block)
    return mask_bucket_batch(np.frombuffer(bytes(block), dtype=np.uint8), [prefix_len])[0].tobytes()


def _count_one(block: bytes, prefix_len: int, symbol: int, kernel: Kernel) -> int:
    _check_bucket(block, prefix_len)
    return int(count_bucket_batch(np.frombuffer(bytes(block), dtype=np.uint8), [prefix_len], [symbol], kernel)[0])


def count_bucket_scalar(block: bytes, prefix_len: int, symbol: int) -> int:
    """kernels.py:137-144 (popcount method)."""
    return _count_one(block, prefix_len, symbol, Kernel.SCALAR)


def count_bucket_bytelut(block: bytes, prefix_len: int, symbol: int) -> int:
    """kernels.py:147-158 (popcount method)."""
    return _count_one(block, prefix_len, symbol, Kernel.BYTELUT)


def count_bucket_nibble(block: bytes, prefix_len: int, symbol: int, trace: KernelTrace | None = None) -> int:
    """kernels.py:161-211: the three-phase half-byte pipeline, on the GPU."""
    _check_bucket(block, prefix_len)
    if trace is None:
        return _count_one(block, prefix_len, symbol, Kernel.NIBBLE)
    t = nibble_trace_batch(np.frombuffer(bytes(block), dtype=np.uint8), [prefix_len], [symbol])[0]
    t = [int(x) for x in t]
    trace.masked_words.extend(t[0:4])
    trace.lookup_lo_words.extend(t[4:8])
    trace.lookup_hi_words.extend(t[8:12])
    trace.group_sads.extend((t[12] >> (16 * g)) & 0xFFFF for g in range(4))
    trace.sad_total = t[13] & 0xFFFFFFFF
    trace.raw_count = t[13] >> 32
    trace.count = t[14]
    return trace.count


def count_bucket_simd(block: bytes, prefix_len: int, symbol: int) -> int:
    """kernels.py:214-228 (nibble pipeline)."""
    return _count_one(block, prefix_len, symbol, Kernel.SIMD)


_COUNT_FNS: dict[Kernel, Callable[[bytes, int, int], int]] = {
    Kernel.SCALAR: count_bucket_scalar,
    Kernel.BYTELUT: count_bucket_bytelut,
    Kernel.NIBBLE: count_bucket_nibble,
    Kernel.SIMD: count_bucket_simd,
    Kernel.GPU: count_bucket_bytelut,
}


def count_fn(kernel: Kernel | str | None = None) -> Callable[[bytes, int, int], int]:
    return _COUNT_FNS[resolve_kernel(kernel)]


def all4_fn(kernel: Kernel | str | None = None) -> Callable[[bytes, int], OccCounts]:
    k = resolve_kernel(kernel)

    def all4(block: bytes, prefix_len: int) -> OccCounts:
        _check_bucket(block, prefix_len)
        return OccCounts(*(int(x) for x in count_bucket_all4_batch(
            np.frombuffer(bytes(block), dtype=np.uint8), [prefix_len], k)[0]))

    return all4


def count_bucket_all4(block: bytes, prefix_len: int, kernel: Kernel | str | None = None) -> OccCounts:
    """All four symbol counts for one bucket prefix (kernels.py:353-358)."""
    _check_bucket(block, prefix_len)
    return all4_fn(kernel)(block, prefix_len)
