"""The reference's acceptance criteria 5-9 (test_acceptance.py:174-285) run
against this package on the GPU, with independent oracles
(tests/acceptance_oracles.py; suffix arrays from the oracle's own build)."""

import numpy as np
import pytest

import paper_1811_06127_b200 as fm
from acceptance_oracles import anchored_edit_distance, hamming_positions, scan_positions
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


@pytest.fixture(scope="module")
def suite5():
    """40 references (10,000 + 39 of 500-10,000 bp) and 1,000 exact cases (test_acceptance.py:60-78)."""
    rng = _rng(105)
    sizes = [10_000] + list(rng.integers(500, 10_001, 39))
    pool = []
    for n in sizes:
        text = rng.integers(0, 4, int(n), dtype=np.uint8)
        pool.append((text, fm.build_index(text)))
    cases = []
    for _ in range(1000):
        rid = int(rng.integers(0, len(pool)))
        text = pool[rid][0]
        m = int(rng.integers(1, 51))
        if rng.random() < 0.7:
            s = int(rng.integers(0, text.size - m + 1))
            pat = text[s:s + m].copy()
        else:
            pat = rng.integers(0, 4, m, dtype=np.uint8)
        cases.append((rid, pat))
    return pool, cases


@pytest.fixture(scope="module")
def suite8():
    """100 references of 100-5,000 bp with their suffix arrays (test_acceptance.py:81-92)."""
    rng = _rng(108)
    out = []
    for _ in range(100):
        text = rng.integers(0, 4, int(rng.integers(100, 5001)), dtype=np.uint8)
        out.append((text, fm.build_index(text), orc.BuiltIndex(text, keep_sa=True).sa.astype(np.int64)))
    return out


def _by_ref(cases):
    groups = {}
    for i, (rid, pat) in enumerate(cases):
        groups.setdefault(rid, []).append((i, pat))
    return groups


def test_criterion5_exact_search_vs_scan(gpu, suite5):
    pool, cases = suite5
    checked = 0
    for rid, items in _by_ref(cases).items():
        text, index = pool[rid]
        pats = ["".join("ACGT"[c] for c in p) for _, p in items]
        kl, _ = fm.exact_search_batch(index, pats)
        lens = np.array([p.size for _, p in items])
        hp, pos, _, _, _, _ = fm.collect_hits_batch(index, np.arange(len(items)), kl[:, 0], kl[:, 1],
                                                    np.zeros(len(items)), lens)
        for j, (_, p) in enumerate(items):
            assert np.array_equal(pos[hp == j], scan_positions(text, p)), (rid, pats[j])
            checked += 1
    assert checked == 1000


def test_criterion6_inexact_soundness(gpu):
    rng = _rng(106)
    hits_checked = 0
    for _ in range(200):
        text = rng.integers(0, 4, int(rng.integers(60, 501)), dtype=np.uint8)
        index = fm.build_index(text)
        m = int(rng.integers(10, 17))
        s = int(rng.integers(0, text.size - m + 1))
        pat = text[s:s + m].copy() if rng.random() < 0.6 else rng.integers(0, 4, m, dtype=np.uint8)
        for z in (1, 2):
            ms = fm.inexact_search_batch(index, pat[None, :], z)
            cnt = np.diff(ms.offsets.astype(np.int64))
            hp, pos, hd, _, _, _ = fm.collect_hits_batch(index, np.repeat(np.arange(1), cnt), ms.k, ms.l,
                                                          ms.diffs, np.array([m]))
            for p_, d_ in zip(pos.tolist(), hd.tolist()):
                assert d_ <= z
                assert anchored_edit_distance(pat, text[p_:p_ + m + z], z) <= z, (pat, z, p_)
                hits_checked += 1
    assert hits_checked > 0


def test_criterion7_completeness_and_zero_budget(gpu, suite5):
    rng = _rng(107)
    for i in range(40):
        z = 1 + (i % 2)
        text = rng.integers(0, 4, int(rng.integers(500, 2001)), dtype=np.uint8)
        index = fm.build_index(text)
        m = int(rng.integers(10, 17))
        start = int(rng.integers(0, text.size - m + 1))
        pat = text[start:start + m].copy()
        for p_ in rng.choice(m, z, replace=False):
            pat[p_] = (pat[p_] + int(rng.integers(1, 4))) % 4
        ms = fm.inexact_search_batch(index, pat[None, :], z)
        cnt = np.diff(ms.offsets.astype(np.int64))
        _, pos, _, _, _, _ = fm.collect_hits_batch(index, np.repeat(np.arange(1), cnt), ms.k, ms.l, ms.diffs,
                                                   np.array([m]))
        reported = set(pos.tolist())
        assert start in reported, (i, z)
        assert set(hamming_positions(text, pat, z).tolist()) <= reported, (i, z)
    pool, cases = suite5
    for rid, items in _by_ref(cases).items():
        _, index = pool[rid]
        pats = ["".join("ACGT"[c] for c in p) for _, p in items]
        kl, _ = fm.exact_search_batch(index, pats)
        ms = fm.inexact_search_batch(index, pats, 0)
        for j in range(len(items)):
            got = ms.results(j)
            if kl[j, 1] < kl[j, 0]:
                assert got == []
            else:
                assert got == [fm.MatchResult(fm.BwmInterval(int(kl[j, 0]), int(kl[j, 1])), 0)]


def test_criterion8_position_recovery(gpu, suite8):
    for _, index, sa in suite8:
        assert np.array_equal(fm.locate_rows(index, np.arange(index.n + 1)), sa)


def test_criterion9_row_sums_and_monotonicity(gpu, suite8):
    for _, index, _ in suite8:
        k = np.arange(index.n + 1)
        occ = fm.occ_pair_batch(index, k, k)[:, 4:].astype(np.int64)
        srow = index.sentinel_row
        assert np.array_equal(occ.sum(axis=1), k + 1 - (srow <= k))
        prev = np.vstack([np.zeros((1, 4), np.int64), occ[:-1]])
        steps = occ - prev
        assert set(np.unique(steps)) <= {0, 1}
        assert np.array_equal(steps.sum(axis=1), np.where(k == srow, 0, 1))
