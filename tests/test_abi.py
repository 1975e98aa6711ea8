"""C-ABI library: loads without a GPU, exports every symbol include/fmgpu.h declares.

No compute calls are made here; on a host without CUDA the product entry
points must raise (there is no CPU fallback).
"""

import ctypes as ct
import re
import subprocess

import numpy as np
import pytest

from conftest import REPO
from paper_1811_06127_b200 import _lib

HEADER = REPO / "include" / "fmgpu.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm[bg]_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("fmg_index_create", "fmg_occ_pair", "fmg_exact", "fmg_inexact", "fmg_locate_rows",
                 "fmb_build", "fmg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_lib.PROTOTYPES)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.lib_path())], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fm[bg]_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_has_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.lib_path())], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_error_channel_and_invalid_args():
    lib = _lib.load()
    # null handle -> FMG_EINVAL, message on the thread-local channel
    rc = lib.fmg_occ_pair(None, None, 0, None, None, None)
    assert rc == _lib.FMG_EINVAL
    assert "null" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    # builder errors map the same way
    rc = lib.fmb_build(None, 0, None, None, None, None, 1)
    assert rc == _lib.FMG_EINVAL and "empty" in _lib.last_error()


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    assert _lib.device_count() == 0
    from paper_1811_06127_b200 import build_index, exact_search, occ_pair_batch

    idx = build_index("ACGTACGTTGCA")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        exact_search(idx, "ACG")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        occ_pair_batch(idx, np.array([0]), np.array([5]))
