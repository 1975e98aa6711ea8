"""The 128-byte chunk layout of HBM-resident indexes (csrc/kernels_chunk.cuh):
every Occ step at every position of small texts (forced on with
FMG_CHUNK_MIN_BYTES=0) and the full config 1-H pair set, against the oracle."""

import numpy as np
import pytest

import paper_1811_06127_b200 as fm
from conftest import small_text
from oracle import oracle as orc
from paper_1811_06127_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("sectors", [2, 4])
@pytest.mark.parametrize("n", [1, 2, 79, 80, 81, 191, 192, 193, 303, 304, 383, 384, 415, 416, 417, 831, 832, 833,
                               5000, 20011])
def test_chunk_layout_every_position(gpu, monkeypatch, n, sectors):
    monkeypatch.setenv("FMG_CHUNK_MIN_BYTES", "0")
    monkeypatch.setenv("FMG_CHUNK_SECTORS", str(sectors))
    text = small_text(n, 7000 + n)
    idx = fm.build_index(text, builder="host")
    assert idx.device_index(0).device_bytes > (n + 1) // 2  # lines + chunks
    ox = orc.OracleIndex(idx)
    p = np.arange(-1, n + 1)
    # every single position, then pairs of every gap class: same sector, same
    # chunk, neighbouring and distant chunks, with k - 1 = -1
    got = fm.occ_pair_batch(idx, p, p)
    assert np.array_equal(got, orc.occ_pair_batch(ox, p, p))
    rng = np.random.Generator(np.random.PCG64(n))
    low = rng.integers(-1, n + 1, 20000)
    high = np.minimum(n, low + rng.choice([0, 1, 5, 40, 112, 300, 416, 900, 5000], 20000))
    assert np.array_equal(fm.occ_pair_batch(idx, low, high), orc.occ_pair_batch(ox, low, high))
    with pytest.raises(ValueError):
        fm.occ_pair_batch(idx, [0], [n + 1])


def test_chunk_layout_device_status(gpu, monkeypatch):
    import torch

    monkeypatch.setenv("FMG_CHUNK_MIN_BYTES", "0")
    n = 3000
    idx = fm.build_index(small_text(n, 77), builder="host")
    kl = torch.tensor([[1, 10], [5, n + 1], [0, n]], dtype=torch.int32, device=gpu)
    with pytest.raises(ValueError):
        fm.occ_pair_batch(idx, kl)  # checked form: raises on the bad pair
    st = torch.zeros(1, dtype=torch.int32, device=gpu)
    out = fm.occ_pair_batch(idx, kl, status=st)  # caller-checked form: asynchronous
    torch.cuda.synchronize()
    assert int(st.item()) == 1
    assert (out[1] == 0).all()
    want = orc.occ_pair_batch(orc.OracleIndex(idx), np.array([0, -1]), np.array([10, n]))
    assert np.array_equal(out[[0, 2]].cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("sectors", [2, 4])
def test_config1h_full_vs_oracle(gpu, monkeypatch, sectors):
    """Config 1-H (1 Gbp text, HBM-resident: chunk layout): all 2^24 bench pairs."""
    monkeypatch.setenv("FMG_CHUNK_SECTORS", str(sectors))
    wl = workloads.config1h()
    idx = fm.build_index(wl.text, builder="gpu")
    got = fm.occ_pair_batch(idx, wl.pairs[:, 0], wl.pairs[:, 1])
    want = orc.occ_pair_batch(orc.OracleIndex(idx), wl.pairs[:, 0], wl.pairs[:, 1])
    assert np.array_equal(got, want)
    idx.release_device()
