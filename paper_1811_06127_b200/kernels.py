"""Kernel selection shim and bucket-level constants.

The reference dispatches every bucket count through a plugin registry
(kernels.py:295-350): Kernel {scalar, bytelut, nibble, simd, auto}, chosen by
argument > FMPM_KERNEL > auto.  Here all counting happens inside the sm_100a
Occ-step kernels (masked popcount over 32-byte lines), so there is exactly one
implementation and no dispatch.  The `kernel=` argument of every public
function is still accepted and validated — an unknown name raises the
reference's ValueError — and then ignored.
"""

from __future__ import annotations

import os
from enum import Enum
from typing import NamedTuple

BUCKET_CHARS = 128
BUCKET_BYTES = 32
ENV_KERNEL = "FMPM_KERNEL"


class OccCounts(NamedTuple):
    """Per-symbol counts in A, C, G, T order (kernels.py:44-50)."""

    a: int
    c: int
    g: int
    t: int


class Kernel(str, Enum):
    SCALAR = "scalar"
    BYTELUT = "bytelut"
    NIBBLE = "nibble"
    SIMD = "simd"
    AUTO = "auto"
    GPU = "gpu"


CONCRETE_KERNELS = (Kernel.GPU,)


def resolve_kernel(kernel: Kernel | str | None = None) -> Kernel:
    """Validate a kernel selection the way the reference does (kernels.py:323-342).

    Every valid name resolves to the GPU kernel; unknown names (argument or
    FMPM_KERNEL) raise ValueError.
    """
    if type(kernel) is Kernel:
        return Kernel.GPU
    if kernel is None:
        kernel = os.environ.get(ENV_KERNEL) or Kernel.AUTO
    try:
        Kernel(kernel)
    except ValueError:
        names = ", ".join(k.value for k in Kernel)
        raise ValueError(f"unknown kernel {kernel!r}; expected one of: {names}") from None
    return Kernel.GPU
