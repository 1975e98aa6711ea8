"""Index-level occurrence queries, served by the sm_100a Occ-step kernel.

Mirrors the reference's occ module (occ.py:1-106) name for name, with the
same arguments, return types and ValueErrors; every count is computed on the
GPU (k_occ_pair through fmg_occ_pair*).  `occ_pair_batch` is the batched
form the scalar functions wrap: one launch for N Occ steps.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from . import _lib
from .device import require_gpu
from .index import FmIndex
from .kernels import Kernel, OccCounts, resolve_kernel

_ZERO = OccCounts(0, 0, 0, 0)


class OccPair(NamedTuple):
    """Occurrence counts at the two positions an interval update needs (occ.py:14-18)."""

    at_low: OccCounts
    at_high: OccCounts


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _torch_stream(device: int) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def validate_pairs(index: FmIndex, low: np.ndarray, high: np.ndarray) -> None:
    """Vectorised form of the reference's position checks (occ.py:44-49, 67-79)."""
    n = index.n
    if (low > high).any():
        i = int(np.flatnonzero(low > high)[0])
        raise ValueError(f"pair positions out of order: {int(low[i])} > {int(high[i])}")
    eq = low == high
    bad_eq = eq & ~((high == -1) | ((high >= 0) & (high <= n)))
    if bad_eq.any():
        i = int(np.flatnonzero(bad_eq)[0])
        raise ValueError(f"position {int(high[i])} outside [-1, {n}]")
    ne = ~eq
    if (ne & (low < -1)).any():
        i = int(np.flatnonzero(ne & (low < -1))[0])
        raise ValueError(f"position {int(low[i])} below -1")
    if (ne & (high > n)).any():
        i = int(np.flatnonzero(ne & (high > n))[0])
        raise ValueError(f"position {int(high[i])} beyond transform end {n}")


def occ_pair_batch(index: FmIndex, low, high=None, kernel: Kernel | str | None = None,
                   device: int | None = None, out=None, status=None):
    """All eight counts for N Occ steps: Occ(b, low[i]) and Occ(b, high[i]).

    Host form: `low`, `high` are integer arrays (low = k-1 may be -1); returns
    an (N, 8) uint32 array [low A, C, G, T, high A, C, G, T].
    Device form: `low` is a CUDA uint32/int32 tensor of shape (N, 2) holding
    (k, l) pairs with k = low + 1 (the kernel's native input); the result is
    an (N, 8) CUDA tensor (uint32 when n >= 2^31, else int32) on torch's
    current stream.  Pairs are validated on the device (k <= l + 1, l <= n)
    into a per-call status word: with `status=None` the call checks it before
    returning (one synchronisation) and raises ValueError like the host form;
    with a caller-supplied int32 CUDA tensor `status` (zeroed by the caller)
    the call stays asynchronous and the caller inspects it (non-zero = error).
    """
    resolve_kernel(kernel)
    if _is_cuda_tensor(low):
        import torch

        kl = low
        if kl.dtype not in (torch.int32, torch.uint32) or kl.dim() != 2 or kl.shape[1] != 2:
            raise ValueError("device pairs must be an (N, 2) int32/uint32 tensor of (k, l)")
        kl = kl.contiguous()
        dev = index.device_index(kl.device.index)
        wide = index.n >= (1 << 31)
        if out is None:
            out = torch.empty((kl.shape[0], 8), dtype=torch.uint32 if wide else torch.int32, device=kl.device)
        elif (not _is_cuda_tensor(out) or out.device != kl.device or not out.is_contiguous()
              or out.dtype not in (torch.int32, torch.uint32) or tuple(out.shape) != (kl.shape[0], 8)):
            raise ValueError("out must be a contiguous (N, 8) int32/uint32 tensor on the pairs' device")
        elif wide and out.dtype != torch.uint32:
            raise ValueError("out must be uint32 when n >= 2^31 (counts exceed int32)")
        check = status is None
        if check:
            status = torch.zeros(1, dtype=torch.int32, device=kl.device)
        elif (not _is_cuda_tensor(status) or status.device != kl.device or status.dtype not in (torch.int32, torch.uint32)
              or status.numel() < 1):
            raise ValueError("status must be an int32/uint32 CUDA tensor on the pairs' device")
        _lib.check(
            _lib.load().fmg_occ_pair(dev.handle, kl.data_ptr(), kl.shape[0], out.data_ptr(), status.data_ptr(),
                                     _torch_stream(dev.device))
        )
        if check and int(status.item()):
            raise ValueError(f"Occ pair out of range or out of order (need k <= l + 1 and l <= {index.n})")
        return out
    low = np.asarray(low, dtype=np.int64).reshape(-1)
    high = np.asarray(high, dtype=np.int64).reshape(-1)
    if low.shape != high.shape:
        raise ValueError("low and high must have the same length")
    validate_pairs(index, low, high)
    kl = np.empty((low.size, 2), dtype=np.uint32)
    # low == high == -1 is occ_all(-1) twice: zeros; encode as k = 0 with l = 0
    # and clear the high half afterwards.
    both_neg = high < 0
    kl[:, 0] = (low + 1).astype(np.uint32)
    kl[:, 1] = np.where(both_neg, 0, high).astype(np.uint32)
    if out is None:
        out = np.empty((low.size, 8), dtype=np.uint32)
    if low.size:
        require_gpu()
        dev = index.device_index(device)
        _lib.check(_lib.load().fmg_occ_pair_host(dev.handle, kl.ctypes.data, low.size, out.ctypes.data))
        if both_neg.any():
            out[both_neg] = 0
    return out


def _one(index: FmIndex, low: int, high: int) -> np.ndarray:
    return occ_pair_batch(index, np.array([low]), np.array([high]))[0]


def occ(index: FmIndex, symbol: int, k: int, kernel: Kernel | str | None = None) -> int:
    """Occurrences of `symbol` in transform rows 0..k inclusive (occ.py:21-41)."""
    if not 0 <= symbol < 4:
        raise ValueError(f"symbol code {symbol} outside [0, 4)")
    if k < 0:
        if k == -1:
            return 0
        raise ValueError(f"position {k} below -1")
    if k > index.n:
        raise ValueError(f"position {k} beyond transform end {index.n}")
    resolve_kernel(kernel)
    return int(_one(index, k, k)[4 + symbol])


def occ_all(index: FmIndex, k: int, kernel: Kernel | str | None = None) -> OccCounts:
    """All four occurrence counts at position k (occ.py:44-56)."""
    if k == -1:
        return _ZERO
    if not 0 <= k <= index.n:
        raise ValueError(f"position {k} outside [-1, {index.n}]")
    resolve_kernel(kernel)
    return OccCounts(*(int(v) for v in _one(index, k, k)[4:]))


def occ_pair_all(index: FmIndex, low: int, high: int, kernel: Kernel | str | None = None) -> OccPair:
    """Counts for all symbols at two positions, low <= high (occ.py:59-96)."""
    if low > high:
        raise ValueError(f"pair positions out of order: {low} > {high}")
    resolve_kernel(kernel)
    if low == high:
        at = occ_all(index, high)
        return OccPair(at_low=at, at_high=at)
    if low < 0 and low != -1:
        raise ValueError(f"position {low} below -1")
    if high > index.n:
        raise ValueError(f"position {high} beyond transform end {index.n}")
    v = _one(index, low, high)
    return OccPair(
        at_low=OccCounts(*(int(x) for x in v[:4])), at_high=OccCounts(*(int(x) for x in v[4:]))
    )


def bwt_char_at(index: FmIndex, i: int) -> int | None:
    """Symbol code at transform row i, None at the sentinel row (occ.py:99-106)."""
    if not 0 <= i <= index.n:
        raise ValueError(f"row {i} outside [0, {index.n}]")
    from .search import psi_inverse_batch

    sym, _ = psi_inverse_batch(index, np.array([i], dtype=np.int64))
    return None if sym[0] == 255 else int(sym[0])
