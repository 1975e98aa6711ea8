"""FM-index host object, native construction and invariant checks.

Mirrors the reference's index module (index.py:12-163): the same fields
(n, c, buckets, sentinel_row, sa_samples, records), the same bucket
semantics ('$' packed as code 0 and counted in the A lane of the bases,
zero-padded last bucket, index.py:24-36, 83-91) and the same errors.  The
difference is storage: buckets live in one numpy array of .fmi bucket
records (B x 64 bytes: 4 x u64 LE base + 32 packed bytes, serialize.py:87-92),
which is what the GPU upload consumes; `buckets` exposes them lazily as
OccBucket tuples for code written against the reference.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .alphabet import encode_array

SA_STRIDE = 32
BUCKET_CHARS = 128
BUCKET_BYTES = 32
RECORD_BYTES = 64


@dataclass(frozen=True)
class RecordSpan:
    """One named stretch of the concatenated reference."""

    name: str
    start: int
    length: int


@dataclass(frozen=True)
class OccBucket:
    """Counter block covering 128 transform characters (index.py:24-36)."""

    base: tuple[int, int, int, int]
    chars: bytes


class _BucketView(Sequence):
    """Read-only sequence of OccBucket over the packed bucket records."""

    def __init__(self, records: np.ndarray):
        self._rec = records
        self._base = records[:, :32].view("<u8")

    def __len__(self) -> int:
        return self._rec.shape[0]

    def __getitem__(self, j):
        if isinstance(j, slice):
            return tuple(self[i] for i in range(*j.indices(len(self))))
        if j < 0:
            j += len(self)
        if not 0 <= j < len(self):
            raise IndexError(j)
        return OccBucket(
            base=tuple(int(x) for x in self._base[j]), chars=self._rec[j, 32:].tobytes()
        )


class FmIndex:
    """Succinct FM-index over a concatenated DNA reference (index.py:39-54).

    Immutable after construction; safe to share across threads.  Device
    copies are created lazily per CUDA device by `device_index()`.
    """

    __slots__ = ("n", "c", "sentinel_row", "records", "bucket_records", "sa_samples", "_dev", "_codes", "_rev")

    def __init__(
        self,
        n: int,
        c: Sequence[int],
        bucket_records: np.ndarray,
        sentinel_row: int,
        sa_samples: np.ndarray,
        records: Sequence[RecordSpan],
    ):
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "c", tuple(int(x) for x in c))
        rec = np.ascontiguousarray(bucket_records, dtype=np.uint8).reshape(-1, RECORD_BYTES)
        rec.setflags(write=False)
        object.__setattr__(self, "bucket_records", rec)
        object.__setattr__(self, "sentinel_row", int(sentinel_row))
        samples = np.ascontiguousarray(sa_samples, dtype=np.uint64)
        samples.setflags(write=False)
        object.__setattr__(self, "sa_samples", samples)
        object.__setattr__(self, "records", tuple(records))
        object.__setattr__(self, "_dev", {})
        object.__setattr__(self, "_codes", None)  # text codes when built here (for the reverse index)
        object.__setattr__(self, "_rev", None)

    def __setattr__(self, name, value):
        raise AttributeError("FmIndex is immutable")

    @property
    def buckets(self) -> _BucketView:
        return _BucketView(self.bucket_records)

    @property
    def bases(self) -> np.ndarray:
        """(B, 4) uint64 bucket bases."""
        return self.bucket_records[:, :32].view("<u8")

    def __eq__(self, other) -> bool:
        if not isinstance(other, FmIndex):
            return NotImplemented
        return (
            self.n == other.n
            and self.c == other.c
            and self.sentinel_row == other.sentinel_row
            and self.records == other.records
            and np.array_equal(self.bucket_records, other.bucket_records)
            and np.array_equal(self.sa_samples, other.sa_samples)
        )

    __hash__ = None

    def __repr__(self) -> str:
        return (
            f"FmIndex(n={self.n}, c={self.c}, buckets={self.bucket_records.shape[0]}, "
            f"sentinel_row={self.sentinel_row}, records={len(self.records)})"
        )

    def reverse_index(self, builder: str = "auto", device: int | None = None) -> tuple[np.ndarray, int]:
        """(bucket records, sentinel row) of the index of the REVERSED text.

        Engine cache for the bidirectional z = 1 search (kernels_bidir.cuh);
        not part of the reference's index or of the .fmi format.  Built from
        the text this index was built from, or from the text recovered from
        the index itself on the GPU (reconstruct_codes: n/32 parallel
        predecessor walks, ~0.3 s at 3.1 Gbp) when it was loaded.
        """
        if self._rev is None:
            codes = self._codes
            if codes is None:  # a loaded index: recover the text on the GPU (k_reconstruct)
                from .search import reconstruct_codes

                codes = reconstruct_codes(self, device)
            rec, _, _, sentinel = _build_arrays(np.ascontiguousarray(codes[::-1]), builder, device, None)
            rec.setflags(write=False)
            object.__setattr__(self, "_rev", (rec, sentinel))
        return self._rev

    def device_index(self, device: int | None = None):
        """The device-resident copy on `device` (created on first use)."""
        from .device import DeviceIndex, current_device

        dev = current_device() if device is None else int(device)
        handle = self._dev.get(dev)
        if handle is None:
            handle = DeviceIndex(self, dev)
            self._dev[dev] = handle
        return handle

    def release_device(self) -> None:
        """Free every device copy of the index."""
        for h in list(self._dev.values()):
            h.close()
        self._dev.clear()


def build_c_table(totals: Sequence[int]) -> tuple[int, int, int, int, int]:
    """Exclusive prefix sums of the four symbol totals (index.py:57-64)."""
    if len(totals) != 4 or any(t < 0 for t in totals):
        raise ValueError("expected four non-negative symbol totals")
    c = [0]
    for t in totals:
        c.append(c[-1] + t)
    return tuple(c)


GPU_BUILD_MIN = 1 << 22  # "auto" builds on the GPU from this many characters up


def build_index(
    reference, records: Sequence[tuple[str, int, int]] | None = None, threads: int | None = None,
    builder: str = "auto", device: int | None = None,
) -> FmIndex:
    """Build the full index for a reference (index.py:67-101), natively.

    `reference` is a DNA string (either case) or an array of codes in [0, 4).
    builder="host": suffix array by SA-IS in C++ (fmb_build); "gpu": prefix
    doubling in HBM (fmb_build_gpu); "auto": the GPU for references of at
    least GPU_BUILD_MIN characters when a CUDA device is visible.  Both give
    identical indexes (the suffix array of text+'$' is unique).
    """
    if builder not in ("auto", "host", "gpu"):
        raise ValueError(f"unknown builder {builder!r}")
    if isinstance(reference, np.ndarray):
        codes = np.ascontiguousarray(reference, dtype=np.uint8)
        if codes.size and codes.max() > 3:
            raise ValueError("symbol code outside [0, 4)")
    else:
        if not reference:
            raise ValueError("reference is empty")
        codes = encode_array(reference)
    n = int(codes.size)
    if n == 0:
        raise ValueError("reference is empty")
    spans = _normalize_records(records, n)
    rec, samples, c, sentinel = _build_arrays(codes, builder, device, threads)
    index = FmIndex(n, c.tolist(), rec, sentinel, samples, spans)
    object.__setattr__(index, "_codes", codes)
    return index


def _build_arrays(codes: np.ndarray, builder: str, device: int | None, threads: int | None):
    """(bucket records, SA samples, C, sentinel row) of text codes + '$'."""
    n = int(codes.size)
    nb = (n + 1 + BUCKET_CHARS - 1) // BUCKET_CHARS
    rec = np.empty((nb, RECORD_BYTES), dtype=np.uint8)
    samples = np.empty(n // SA_STRIDE + 1, dtype=np.uint64)
    c = np.zeros(5, dtype=np.uint64)
    sentinel = np.zeros(1, dtype=np.uint64)
    lib = _lib.load()
    auto = builder == "auto"
    if auto:
        builder = "gpu" if n >= GPU_BUILD_MIN and _lib.device_count() > 0 else "host"
    if builder == "gpu":
        from .device import current_device, require_gpu

        require_gpu()
        dev = current_device() if device is None else int(device)
        status = lib.fmb_build_gpu(
            dev, codes.ctypes.data, n, rec.ctypes.data, samples.ctypes.data, c.ctypes.data,
            sentinel.ctypes.data, None,
        )
        if auto and status != _lib.FMG_OK and "out of memory" in _lib.last_error():
            # the GPU builder wants ~36 bytes per character of device memory; when search
            # tables already hold it (a reverse index built late), the host builder does the job
            builder = "host"
        else:
            _lib.check(status)
    if builder != "gpu":
        _lib.check(
            lib.fmb_build(
                codes.ctypes.data, n, rec.ctypes.data, samples.ctypes.data, c.ctypes.data,
                sentinel.ctypes.data, int(threads or os.cpu_count() or 1),
            )
        )
    return rec, samples, c, int(sentinel[0])


def suffix_array(reference) -> np.ndarray:
    """Suffix array of reference + '$' (uint32, length n+1), via native SA-IS."""
    codes = (
        np.ascontiguousarray(reference, dtype=np.uint8)
        if isinstance(reference, np.ndarray)
        else encode_array(reference)
    )
    if codes.size == 0:
        raise ValueError("reference is empty")
    sa = np.empty(codes.size + 1, dtype=np.uint32)
    _lib.check(_lib.load().fmb_suffix_array(codes.ctypes.data, codes.size, sa.ctypes.data))
    return sa


def _normalize_records(
    records: Sequence[tuple[str, int, int]] | None, n: int
) -> tuple[RecordSpan, ...]:
    """index.py:104-122: records must tile [0, n) contiguously."""
    if records is None:
        return (RecordSpan(name="ref", start=0, length=n),)
    spans = []
    expected_start = 0
    for name, start, length in records:
        if not name:
            raise ValueError("record name is empty")
        if start != expected_start or length <= 0:
            raise ValueError(
                f"record {name!r} (start={start}, length={length}) does not tile the reference"
            )
        spans.append(RecordSpan(name=name, start=start, length=length))
        expected_start = start + length
    if expected_start != n:
        raise ValueError(f"records cover {expected_start} of {n} characters")
    return tuple(spans)


def _bucket_counts(records: np.ndarray, prefix: np.ndarray) -> np.ndarray:
    """(B, 4) counts of each code among the first prefix[j] fields of bucket j."""
    chars = records[:, 32:]
    fields = np.stack([(chars >> s) & 3 for s in (0, 2, 4, 6)], axis=-1).reshape(len(records), 128)
    live = np.arange(128)[None, :] < prefix[:, None]
    return np.stack([((fields == s) & live).sum(axis=1) for s in range(4)], axis=1)


def check_index(index: FmIndex) -> None:
    """Validate structural invariants (index.py:125-163); ValueError on violation."""
    n = index.n
    if n <= 0:
        raise ValueError("index covers an empty reference")
    if index.c[0] != 0 or index.c[4] != n:
        raise ValueError(f"C table endpoints wrong: {index.c}")
    if any(a > b for a, b in zip(index.c, index.c[1:])):
        raise ValueError(f"C table not non-decreasing: {index.c}")
    nb = index.bucket_records.shape[0]
    expected_buckets = (n + 1 + BUCKET_CHARS - 1) // BUCKET_CHARS
    if nb != expected_buckets:
        raise ValueError(f"expected {expected_buckets} buckets for n={n}, found {nb}")
    if not 0 <= index.sentinel_row <= n:
        raise ValueError(f"sentinel row {index.sentinel_row} outside [0, {n}]")
    if len(index.sa_samples) != n // SA_STRIDE + 1:
        raise ValueError(f"expected {n // SA_STRIDE + 1} samples, found {len(index.sa_samples)}")
    if len(index.sa_samples) and int(index.sa_samples.max()) > n:
        raise ValueError("suffix-array sample out of range")
    inside_len = np.minimum(BUCKET_CHARS, n + 1 - np.arange(nb, dtype=np.int64) * BUCKET_CHARS)
    inside = _bucket_counts(index.bucket_records, inside_len)
    full = _bucket_counts(index.bucket_records, np.full(nb, BUCKET_CHARS))
    expect = np.zeros((nb, 4), dtype=np.uint64)
    np.cumsum(inside[:-1].astype(np.uint64), axis=0, out=expect[1:])
    bad = np.flatnonzero((index.bases != expect).any(axis=1))
    if bad.size:
        j = int(bad[0])
        raise ValueError(
            f"bucket {j} base {tuple(int(x) for x in index.bases[j])} breaks telescoping "
            f"({tuple(int(x) for x in expect[j])})"
        )
    pad = full - inside
    pad_bad = (pad[:, 0] != BUCKET_CHARS - inside_len) | (pad[:, 1:] != 0).any(axis=1)
    if pad_bad.any():
        raise ValueError(f"bucket {int(np.flatnonzero(pad_bad)[0])} padding fields are not zero")
    _normalize_records([(r.name, r.start, r.length) for r in index.records], n)
