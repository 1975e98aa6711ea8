"""Device-resident index handle (fmg_index) and device selection."""

from __future__ import annotations

import ctypes as ct
import threading

import numpy as np

from . import _lib


def current_device() -> int:
    """torch's current CUDA device when torch is in use, else device 0."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    return 0


def require_gpu() -> None:
    """Fail loudly when there is no CUDA device: there is no CPU fallback."""
    if _lib.device_count() == 0:
        raise RuntimeError(
            "no CUDA device visible: the fmgpu engine runs only on the GPU (no CPU fallback)"
        )


class DeviceIndex:
    """Owns one fmg_index: the index re-laid out as 32-byte lines in HBM.

    Upload cost is paid once per (index, device); the handle is immutable and
    may be used from several threads/streams concurrently.
    """

    def __init__(self, index, device: int):
        require_gpu()
        lib = _lib.load()
        c = np.asarray(index.c, dtype=np.uint64)
        self._c = c
        handle = ct.c_void_p()
        _lib.check(
            lib.fmg_index_create(
                int(device), index.bucket_records.ctypes.data, index.bucket_records.shape[0],
                index.n, index.sentinel_row, c.ctypes.data, ct.byref(handle),
            )
        )
        self.handle = handle
        self.device = int(device)
        self.n = index.n
        self._has_samples = False
        self._has_reverse = False
        self._index = index
        # one-time attachments: check-then-act under a lock (the C side is
        # also idempotent and never frees an attached buffer before destroy)
        self._attach = threading.RLock()  # ensure_reverse may need ensure_samples (text recovery)

    def ensure_reverse(self) -> None:
        """Attach the reversed-text index (bidirectional z = 1 engine)."""
        with self._attach:
            if not self._has_reverse:
                rec, sentinel = self._index.reverse_index(device=self.device)
                _lib.check(_lib.load().fmg_index_set_reverse(self.handle, rec.ctypes.data, rec.shape[0], sentinel))
                self._has_reverse = True

    def wants_reverse(self, count: int, max_len: int, max_diff: int) -> bool:
        """Whether a bounded-difference batch of this shape would read a reverse index
        (fmg_inexact_wants_reverse: the bidirectional z = 1 engines do, the flat engine of
        HBM-resident indexes and every other engine do not)."""
        wants = ct.c_int()
        _lib.check(_lib.load().fmg_inexact_wants_reverse(self.handle, int(count), int(max_len), int(max_diff),
                                                         ct.byref(wants)))
        return bool(wants.value)

    def ensure_samples(self) -> None:
        if self._has_samples:
            return
        with self._attach:
            if not self._has_samples:
                s = self._index.sa_samples
                _lib.check(_lib.load().fmg_index_set_samples(self.handle, s.ctypes.data, s.size))
                self._has_samples = True

    @property
    def device_bytes(self) -> int:
        nb = ct.c_uint64()
        _lib.check(_lib.load().fmg_index_info(self.handle, None, None, ct.byref(nb)))
        return nb.value

    def close(self) -> None:
        if self.handle:
            _lib.load().fmg_index_destroy(self.handle)
            self.handle = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
