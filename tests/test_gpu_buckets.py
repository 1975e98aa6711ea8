"""Bucket-level GPU kernels (csrc/kernels_bucket.cuh) against the reference:
the paper's Figure 2 known answers, the reference's kernel tests and
acceptance criteria 2-4 (test_kernels.py:51-180, test_acceptance.py:113-172),
and the reference's own answers on 3,000 seeded buckets (tests/golden)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import bucket_oracle as bo
from paper_1811_06127_b200 import kernels as K
from paper_1811_06127_b200 import pack_2bit, pack_codes

pytestmark = pytest.mark.gpu

FIG_STRING = "ccacttgcgaaatttacaaggtttattaggtt"
FIG_BLOCK = pack_2bit(FIG_STRING).data + bytes(32 - 8)
COUNT_FNS = [K.count_bucket_scalar, K.count_bucket_bytelut, K.count_bucket_nibble, K.count_bucket_simd]


def test_figure2_packed_block_and_trace(gpu):
    # test_acceptance.py:113-121 (criterion 2), test_kernels.py:89-107
    assert int.from_bytes(pack_2bit(FIG_STRING).data, "little") == 0xFA3CFE813F026F45
    tr = K.KernelTrace()
    assert K.count_bucket_nibble(FIG_BLOCK, 32, 2, trace=tr) == 6
    assert tr.masked_words[0] == 0xFA3CFE813F026F45
    assert tr.lookup_lo_words[0] == 0xDFBEAFFA7FEE7FF7
    assert tr.lookup_hi_words[0] == 0x8041801141021405
    assert tr.group_sads == [0x7F2, 2040, 2040, 2040]
    assert tr.sad_total == 0x7F2 + 3 * 2040
    assert tr.raw_count == 8160 - tr.sad_total == 6
    assert tr.count == 6


def test_figure2_counts(gpu):
    # test_kernels.py:62-66, 157-159
    for fn in COUNT_FNS:
        assert fn(FIG_BLOCK, 32, 2) == 6
        assert fn(FIG_BLOCK, 7, 2) == 1
        assert fn(FIG_BLOCK, 0, 2) == 0
        assert fn(FIG_BLOCK, 32, 3) == 12
    for kern in K.CONCRETE_KERNELS:
        assert tuple(K.count_bucket_all4(FIG_BLOCK, 32, kern)) == (9, 5, 6, 12)


def test_zero_partial_and_mask(gpu):
    # test_kernels.py:51-75, 173-180
    zero = bytes(32)
    for fn in COUNT_FNS:
        assert fn(zero, 128, 0) == 128
        assert fn(zero, 0, 0) == 0
        assert fn(zero, 128, 1) == 0
        assert fn(zero, 77, 0) == 77
    block = pack_codes([2, 0, 1, 0, 0], pad_to=32)
    for fn in COUNT_FNS:
        assert [fn(block, 5, s) for s in range(4)] == [3, 1, 1, 0]
    ff = bytes([0xFF] * 32)
    assert K.mask_bucket(ff, 0) == bytes(32)
    assert K.mask_bucket(ff, 128) == ff
    m = K.mask_bucket(ff, 5)
    assert m[0] == 0xFF and m[1] == 0x03 and set(m[2:]) == {0}


def test_reference_answers_on_seeded_buckets(gpu):
    g = dict(np.load(GOLDEN / "buckets.npz"))
    b, pl, sy = g["blocks"], g["prefix"], g["symbol"]
    for kern in K.CONCRETE_KERNELS:
        assert np.array_equal(K.count_bucket_batch(b, pl, sy, kern), g["counts"][:, 0]), kern
        assert np.array_equal(K.count_bucket_all4_batch(b, pl, kern), g["all4"]), kern
    assert np.array_equal(K.mask_bucket_batch(b, pl), g["masked"])
    assert np.array_equal(K.nibble_trace_batch(b, pl, sy), g["trace"])


def test_criterion3_kernel_equivalence(gpu):
    # test_acceptance.py:124-156: 100,000 random buckets / prefixes / symbols,
    # then every prefix length of 100 buckets, both GPU methods vs the scalar oracle
    rng = np.random.Generator(np.random.PCG64(103))
    n = 100_000
    blocks = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    pl = rng.integers(0, 129, n)
    sy = rng.integers(0, 4, n)
    want = bo.count_scalar(blocks, pl, sy)
    for kern in ("bytelut", "nibble"):
        assert np.array_equal(K.count_bucket_batch(blocks, pl, sy, kern), want), kern
    sweep = np.repeat(rng.integers(0, 256, (100, 32), dtype=np.uint8), 129, axis=0)
    spl = np.tile(np.arange(129), 100)
    ssy = rng.integers(0, 4, sweep.shape[0])
    want = bo.count_scalar(sweep, spl, ssy)
    want4 = bo.all4_scalar(sweep, spl)
    for kern in ("scalar", "simd"):
        assert np.array_equal(K.count_bucket_batch(sweep, spl, ssy, kern), want), kern
        assert np.array_equal(K.count_bucket_all4_batch(sweep, spl, kern), want4), kern


def test_criterion4_sad_identity_and_monotone(gpu):
    # test_acceptance.py:159-172, test_kernels.py:110-119, 162-170
    rng = np.random.Generator(np.random.PCG64(104))
    blocks = np.repeat(rng.integers(0, 256, (120, 32), dtype=np.uint8), 4, axis=0)
    sy = np.tile(np.arange(4), 120)
    tr = K.nibble_trace_batch(blocks, np.full(480, 128), sy)
    total, raw = tr[:, 13] & 0xFFFFFFFF, tr[:, 13] >> 32
    assert np.array_equal(raw, 8160 - total)
    assert np.array_equal(tr[:, 14], raw)  # full bucket: no padding correction
    assert np.array_equal(tr[:, 14], bo.count_scalar(blocks, np.full(480, 128), sy))
    one = np.repeat(rng.integers(0, 256, (1, 32), dtype=np.uint8), 129 * 4, axis=0)
    c = K.count_bucket_batch(one, np.repeat(np.arange(129), 4), np.tile(np.arange(4), 129), "nibble")
    d = np.diff(c.reshape(129, 4).astype(np.int64), axis=0)
    assert set(np.unique(d)) <= {0, 1} and (d.sum(axis=1) == 1).all()


def test_device_form_and_status(gpu):
    import torch

    from paper_1811_06127_b200 import _lib

    rng = np.random.Generator(np.random.PCG64(9))
    blocks = rng.integers(0, 256, (1000, 32), dtype=np.uint8)
    pl = rng.integers(0, 129, 1000).astype(np.uint32)
    pl[7] = 300  # bad prefix: reported through the caller's status word, zeros written
    d_b = torch.from_numpy(blocks).cuda()
    d_pl = torch.from_numpy(pl.view(np.int32)).cuda()
    out = torch.empty((1000, 4), dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().fmg_bucket_count(d_b.data_ptr(), d_pl.data_ptr(), None, 1000, 1, out.data_ptr(),
                                            st.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(st.item()) == 1
    got = out.cpu().numpy()
    ok = np.arange(1000) != 7
    assert np.array_equal(got[ok], bo.all4_scalar(blocks[ok], pl[ok]))
    assert (got[7] == 0).all()
