"""Compile the in-tree native library (libfmgpu.so) for sm_100a.

The library holds the CUDA kernels, the C ABI of include/fmgpu.h and the
native index builder.  It is built in-tree so it travels with the repository
snapshot to the GPU box; nvcc cross-compiles without a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libfmgpu.so"

SOURCES = ["fmgpu.cu", "build_gpu.cu", "builder.cpp"]
HEADERS = ["fmgpu_internal.h", "occ_device.cuh", "kernels_occ.cuh", "kernels_search.cuh", "kernels_inexact.cuh",
           "kernels_bidir.cuh", "kernels_flat.cuh", "kernels_bucket.cuh", "kernels_chunk.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
    "-ldl",  # guard mode resolves the driver API (libcuda) at run time: no link-time dependency
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfmgpu.so")


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [REPO_DIR / "include" / "fmgpu.h"]
    return any(p.stat().st_mtime > built for p in deps)


def build_native(force: bool = False, verbose: bool = False, out: Path | None = None,
                 extra: list[str] | None = None) -> Path:
    """Build libfmgpu.so if any source is newer than the library.

    `out` / `extra` (extra nvcc flags, e.g. -D switches) are for A/B variant
    builds only (tools/ab/); the package always loads LIB_PATH.
    """
    target = Path(out) if out else LIB_PATH
    if out is None and not force and not _stale():
        return LIB_PATH
    tmp = target.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, *(extra or []), "-I", str(REPO_DIR / "include"),
           *[str(CSRC / s) for s in SOURCES], "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    import sys

    # python -m paper_1811_06127_b200._build [out.so -DFLAG ...]   (variant builds for A/B)
    args = sys.argv[1:]
    print(build_native(force=True, verbose=True, out=Path(args[0]).resolve() if args else None, extra=args[1:]))
