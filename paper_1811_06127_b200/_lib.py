"""ctypes binding of libfmgpu.so (include/fmgpu.h).

There is no CPU fallback: if the library is missing this module raises on
first use, and every search/Occ entry point needs a CUDA device.
"""

from __future__ import annotations

import ctypes as ct
import os
import threading
from pathlib import Path

from ._build import LIB_PATH

FMG_OK, FMG_EINVAL, FMG_ECAPACITY, FMG_ECUDA, FMG_ENOMEM, FMG_EINTERNAL = range(6)

_u8p = ct.POINTER(ct.c_uint8)
_u32p = ct.POINTER(ct.c_uint32)
_u64p = ct.POINTER(ct.c_uint64)
_vp = ct.c_void_p

# name -> (restype, argtypes); every symbol include/fmgpu.h declares
PROTOTYPES: dict[str, tuple] = {
    "fmg_last_error": (ct.c_char_p, []),
    "fmg_device_count": (ct.c_int, [ct.POINTER(ct.c_int)]),
    "fmb_suffix_array": (ct.c_int, [_vp, ct.c_uint64, _vp]),
    "fmb_build": (ct.c_int, [_vp, ct.c_uint64, _vp, _vp, _vp, _vp, ct.c_int]),
    "fmb_build_gpu": (ct.c_int, [ct.c_int, _vp, ct.c_uint64, _vp, _vp, _vp, _vp, _vp]),
    "fmg_index_create": (ct.c_int, [ct.c_int, _vp, ct.c_uint64, ct.c_uint64, ct.c_uint64, _vp,
                                    ct.POINTER(_vp)]),
    "fmg_index_set_samples": (ct.c_int, [_vp, _vp, ct.c_uint64]),
    "fmg_index_set_reverse": (ct.c_int, [_vp, _vp, ct.c_uint64, ct.c_uint64]),
    "fmg_index_has_reverse": (ct.c_int, [_vp, ct.POINTER(ct.c_int)]),
    "fmg_index_info": (ct.c_int, [_vp, _u64p, ct.POINTER(ct.c_int), _u64p]),
    "fmg_index_destroy": (None, [_vp]),
    "fmg_occ_pair": (ct.c_int, [_vp, _vp, ct.c_uint64, _vp, _vp, _vp]),
    "fmg_occ_pair_host": (ct.c_int, [_vp, _vp, ct.c_uint64, _vp]),
    "fmg_exact": (ct.c_int, [_vp, _vp, _vp, ct.c_uint64, _vp, _vp]),
    "fmg_exact_packed": (ct.c_int, [_vp, _vp, ct.c_uint32, ct.c_uint64, _vp, _vp]),
    "fmg_exact_host": (ct.c_int, [_vp, _vp, _vp, ct.c_uint64, _vp]),
    "fmg_exact_packed_host": (ct.c_int, [_vp, _vp, ct.c_uint32, ct.c_uint64, _vp]),
    "fmg_inexact": (ct.c_int, [_vp, _vp, _vp, ct.c_uint64, ct.c_int, ct.POINTER(_vp), _vp]),
    "fmg_inexact_host": (ct.c_int, [_vp, _vp, _vp, ct.c_uint64, ct.c_int, ct.POINTER(_vp)]),
    "fmg_inexact_wants_reverse": (ct.c_int, [_vp, ct.c_uint64, ct.c_uint64, ct.c_int, ct.POINTER(ct.c_int)]),
    "fmg_inexact_packed": (ct.c_int, [_vp, _vp, ct.c_uint32, ct.c_uint64, ct.c_int, ct.POINTER(_vp), _vp]),
    "fmg_inexact_packed_host": (ct.c_int, [_vp, _vp, ct.c_uint32, ct.c_uint64, ct.c_int, ct.POINTER(_vp)]),
    "fmg_matches_size": (ct.c_int, [_vp, _u64p, _u64p]),
    "fmg_matches_steps": (ct.c_int, [_vp, _u64p]),
    "fmg_matches_copy": (ct.c_int, [_vp, _vp, _vp, _vp, _vp, ct.c_int]),
    "fmg_matches_free": (None, [_vp]),
    "fmg_psi_inverse": (ct.c_int, [_vp, _vp, ct.c_uint64, _vp, _vp, _vp, _vp]),
    "fmg_locate_rows": (ct.c_int, [_vp, _vp, ct.c_uint64, _vp, _vp, _vp]),
    "fmg_locate_rows_host": (ct.c_int, [_vp, _vp, ct.c_uint64, _vp]),
    "fmg_reconstruct_text": (ct.c_int, [_vp, _vp, _vp, _vp]),
    "fmg_reconstruct_text_host": (ct.c_int, [_vp, _vp]),
    "fmg_bucket_count": (ct.c_int, [_vp, _vp, _vp, ct.c_uint64, ct.c_int, _vp, _vp, _vp]),
    "fmg_bucket_count_host": (ct.c_int, [ct.c_int, _vp, _vp, _vp, ct.c_uint64, ct.c_int, _vp]),
    "fmg_bucket_mask_host": (ct.c_int, [ct.c_int, _vp, _vp, ct.c_uint64, _vp]),
    "fmg_bucket_nibble_trace_host": (ct.c_int, [ct.c_int, _vp, _vp, _vp, ct.c_uint64, _vp]),
    "fmg_stream_sync": (ct.c_int, [_vp]),
}

_lock = threading.Lock()
_lib: ct.CDLL | None = None


def lib_path() -> Path:
    """The library to load; FMG_LIB_PATH overrides it (A/B experiments only)."""
    return Path(os.environ.get("FMG_LIB_PATH", LIB_PATH))


def load() -> ct.CDLL:
    """Load libfmgpu.so once; raises RuntimeError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = lib_path()
            if not path.exists():
                raise RuntimeError(
                    f"native library {path} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ct.CDLL(str(path))
            for name, (res, args) in PROTOTYPES.items():
                if path != LIB_PATH and not hasattr(lib, name):
                    continue  # an older build under A/B test
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().fmg_last_error().decode("utf-8", "replace")


def check(status: int, what: str = "") -> None:
    """Map an fmg_status to the exception the reference raises."""
    if status == FMG_OK:
        return
    msg = last_error() or what
    if status == FMG_EINVAL:
        raise ValueError(msg)
    if status == FMG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"fmgpu: {msg}")


def device_count() -> int:
    n = ct.c_int(0)
    check(load().fmg_device_count(ct.byref(n)))
    return n.value


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
