"""Bucket-level surface without a GPU: the oracle's restatement of the
reference kernels pinned to the reference's own outputs, the host-side
argument checks, kernel selection and the nibble tables (kernels.py:53-358)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import bucket_oracle as bo
from paper_1811_06127_b200 import kernels as K


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLDEN / "buckets.npz"))


def test_oracle_counts_match_reference(gold):
    want = gold["counts"]  # scalar, bytelut, nibble, simd answers of the reference
    assert (want == want[:, :1]).all()
    got = bo.count_scalar(gold["blocks"], gold["prefix"], gold["symbol"])
    assert np.array_equal(got, want[:, 0])
    assert np.array_equal(bo.all4_scalar(gold["blocks"], gold["prefix"]), gold["all4"])


def test_oracle_mask_and_trace_match_reference(gold):
    assert np.array_equal(bo.mask(gold["blocks"], gold["prefix"]), gold["masked"])
    assert np.array_equal(bo.nibble_trace(gold["blocks"], gold["prefix"], gold["symbol"]), gold["trace"])


def test_nibble_tables(gold):
    # kernels.py:53-77; test_kernels.py:36-46
    t = K.NibbleTables.build()
    assert t == K.TABLES
    assert np.array_equal(np.frombuffer(t.lo, np.uint8), gold["tables_lo"])
    assert np.array_equal(np.frombuffer(t.hi, np.uint8), gold["tables_hi"])
    lo, hi = bo.tables()
    assert lo.tobytes() == t.lo and hi.tobytes() == t.hi
    for v in range(16):
        assert sum((t.hi[v] >> (2 * s)) & 3 for s in range(4)) == 2
        assert t.lo[v] == (~t.hi[v]) & 0xFF


def test_figure2_oracle_trace():
    # test_kernels.py:26-27, 89-107; test_acceptance.py:113-121 (the paper's Figure 2)
    from paper_1811_06127_b200 import pack_2bit

    block = np.frombuffer(pack_2bit("ccacttgcgaaatttacaaggtttattaggtt").data + bytes(24), dtype=np.uint8)
    tr = bo.nibble_trace(block[None, :], [32], [2])[0]
    assert int(tr[0]) == 0xFA3CFE813F026F45
    assert int(tr[4]) == 0xDFBEAFFA7FEE7FF7
    assert int(tr[8]) == 0x8041801141021405
    assert [(int(tr[12]) >> (16 * g)) & 0xFFFF for g in range(4)] == [0x7F2, 2040, 2040, 2040]
    assert int(tr[14]) == 6
    assert tuple(bo.all4_scalar(block[None, :], [32])[0]) == (9, 5, 6, 12)
    assert int(bo.count_scalar(block[None, :], [7], [2])[0]) == 1


def test_bad_arguments_rejected_before_the_gpu():
    # test_kernels.py:77-86: every count function validates its bucket first
    zero = bytes(32)
    for fn in (K.count_bucket_scalar, K.count_bucket_bytelut, K.count_bucket_nibble, K.count_bucket_simd):
        with pytest.raises(ValueError):
            fn(zero[:-1], 4, 0)
        with pytest.raises(ValueError):
            fn(zero, 129, 0)
        with pytest.raises(ValueError):
            fn(zero, -1, 0)
    with pytest.raises(ValueError):
        K.count_bucket_batch(np.zeros((2, 32), np.uint8), [1], [0])
    with pytest.raises(ValueError):
        K.count_bucket_batch(np.zeros((1, 32), np.uint8), [1], [4])
    with pytest.raises(ValueError):
        K.count_bucket_all4_batch(np.zeros((1, 32), np.uint8), [200])


def test_resolve_kernel_like_the_reference(monkeypatch):
    # test_kernels.py:183-196
    assert K.resolve_kernel("scalar") is K.Kernel.SCALAR
    assert K.resolve_kernel(K.Kernel.NIBBLE) is K.Kernel.NIBBLE
    assert K.resolve_kernel("auto") is K.Kernel.BYTELUT
    monkeypatch.delenv("FMPM_KERNEL", raising=False)
    assert K.resolve_kernel(None) is K.Kernel.BYTELUT
    monkeypatch.setenv("FMPM_KERNEL", "simd")
    assert K.resolve_kernel(None) is K.Kernel.SIMD
    monkeypatch.setenv("FMPM_KERNEL", "bogus")
    with pytest.raises(ValueError, match="unknown kernel"):
        K.resolve_kernel(None)
    with pytest.raises(ValueError):
        K.resolve_kernel("avx999")
    assert K.count_fn("scalar") is K.count_bucket_scalar
    assert K.count_fn("nibble") is K.count_bucket_nibble
    assert set(K.CONCRETE_KERNELS) == {K.Kernel.SCALAR, K.Kernel.BYTELUT, K.Kernel.NIBBLE, K.Kernel.SIMD}
