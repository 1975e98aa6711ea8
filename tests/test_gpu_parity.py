"""GPU parity: the sm_100a path vs the reference's outputs and the CPU oracle.

Every comparison is bit-exact (integer work).  Known-answer values are the
reference tests' own (cited); fixtures come from the reference itself
(tests/golden/make_golden.py); large cases compare against the oracle,
which test_oracle.py pins to those fixtures.
"""

import hashlib
import json

import numpy as np
import pytest

import paper_1811_06127_b200 as fm
from conftest import GOLDEN, codes_to_str, small_text
from oracle import oracle as orc
from paper_1811_06127_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acag(gpu):
    return fm.build_index("ACAG")


ACAG_OCC = [(0, 0, 1, 0), (0, 0, 1, 0), (0, 1, 1, 0), (1, 1, 1, 0), (2, 1, 1, 0)]


def test_acag_occ_api(acag):
    # reference tests/test_occ.py:28-99
    for k, row in enumerate(ACAG_OCC):
        for s in range(4):
            assert fm.occ(acag, s, k) == row[s]
        assert tuple(fm.occ_all(acag, k)) == row
    assert fm.occ(acag, 0, -1) == 0
    with pytest.raises(ValueError):
        fm.occ(acag, 0, 5)
    with pytest.raises(ValueError):
        fm.occ(acag, 0, -2)
    with pytest.raises(ValueError):
        fm.occ(acag, 4, 0)
    p = fm.occ_pair_all(acag, 2, 4)
    assert tuple(p.at_low) == (0, 1, 1, 0) and tuple(p.at_high) == (2, 1, 1, 0)
    p = fm.occ_pair_all(acag, -1, 4)
    assert tuple(p.at_low) == (0, 0, 0, 0) and tuple(p.at_high) == (2, 1, 1, 0)
    p = fm.occ_pair_all(acag, 3, 3)
    assert p.at_low == p.at_high
    with pytest.raises(ValueError):
        fm.occ_pair_all(acag, 3, 2)
    assert [fm.bwt_char_at(acag, i) for i in range(5)] == [2, None, 1, 0, 0]
    with pytest.raises(ValueError):
        fm.bwt_char_at(acag, 5)


def test_acag_search_api(acag):
    # reference tests/test_search.py:33-153, 200-249
    B = fm.BwmInterval
    assert fm.init_interval(acag, 0) == B(1, 2)
    assert fm.init_interval(acag, 3) == B(5, 4)
    assert fm.extend_backward(acag, B(1, 2), 1) == B(3, 3)
    assert fm.extend_backward(acag, B(4, 4), 0) == B(2, 2)
    with pytest.raises(ValueError):
        fm.extend_backward(acag, B(5, 4), 0)
    assert fm.exact_search(acag, "CA") == B(3, 3)
    assert fm.exact_search(acag, "ACAG") == B(1, 1)
    assert fm.exact_search(acag, "T").is_empty and fm.exact_search(acag, "GG").is_empty
    r = fm.exact_search(acag, "ANG")
    assert r.is_empty and r.degenerate
    with pytest.raises(ValueError):
        fm.exact_search(acag, "")
    assert fm.inexact_search(acag, "AG", 0) == [fm.MatchResult(B(2, 2), 0)]
    assert fm.inexact_search(acag, "T", 0) == []
    hits, _ = fm.collect_hits(acag, fm.inexact_search(acag, "AT", 1), 2)
    assert [(h.global_pos, h.diffs) for h in hits] == [(0, 1), (2, 1)]
    assert fm.inexact_search(acag, "TT", 2) and fm.inexact_search(acag, "T", 1)
    with pytest.raises(ValueError):
        fm.inexact_search(acag, "A", -1)
    assert fm.inexact_search(acag, "AN", 1) == []
    assert fm.psi_inverse(acag, 2) == 3 and fm.psi_inverse(acag, 4) == 2
    assert fm.psi_inverse(acag, 0) == 4 and fm.psi_inverse(acag, 1) is None
    assert fm.psi_inverse_fused(acag, 2) == (1, 3)
    with pytest.raises(ValueError):
        fm.psi_inverse(acag, 5)
    assert [fm.locate_row(acag, i) for i in range(5)] == [4, 0, 2, 1, 3]
    assert fm.locate_all(acag, B(5, 4), 0, 1) == []


def test_records_and_hits(gpu):
    # reference tests/test_search.py:243-283
    idx = fm.build_index("AAACCC" + "GGGTTT", [("r1", 0, 6), ("r2", 6, 6)])
    hits = fm.locate_all(idx, fm.exact_search(idx, "CCC"), 0, 3)
    assert hits == [fm.Hit(record="r1", offset=3, global_pos=3, diffs=0)]
    iv = fm.exact_search(idx, "CCGG")
    assert not iv.is_empty and fm.locate_all(idx, iv, 0, 4) == []
    idx = fm.build_index("AC" * 50)
    iv = fm.exact_search(idx, "AC")
    hits, trunc = fm.collect_hits(idx, [fm.MatchResult(iv, 0)], 2, max_hits=10)
    assert trunc and len(hits) == 10
    hits, trunc = fm.collect_hits(idx, [fm.MatchResult(iv, 0)], 2)
    assert not trunc and len(hits) == 50
    idx = fm.build_index("ACGTACGTAC")
    hits, _ = fm.collect_hits(idx, fm.inexact_search(idx, "ACGT", 1), 4)
    by = {h.global_pos: h.diffs for h in hits}
    assert by[0] == 0 and by[4] == 0


def test_reconstruct_round_trip(gpu):
    for n in (1, 5, 127, 128, 129, 500):
        codes = small_text(n, 62 + n)
        assert fm.reconstruct_reference(fm.build_index(codes)) == codes_to_str(codes)


def test_small_cases_all_paths(small_cases, gpu):
    for key, case in small_cases.items():
        n = case["n"]
        idx = fm.build_index(small_text(n, case["seed"]))
        occ = fm.occ_pair_batch(idx, case["occ_low"], case["occ_high"])
        assert np.array_equal(occ.astype(np.int64), np.array(case["occ"])), key
        kl, deg = fm.exact_search_batch(idx, case["exact_patterns"])
        assert np.array_equal(kl, np.array(case["exact_kl"])) and not deg.any(), key
        # packed fixed-length path on the same patterns, grouped by length
        pats = case["exact_patterns"]
        for m in sorted({len(p) for p in pats}):
            sel = [i for i, p in enumerate(pats) if len(p) == m]
            if m > 32:
                continue
            arr = np.array([[ "ACGT".index(ch) for ch in pats[i]] for i in sel], dtype=np.uint8)
            klp, _ = fm.exact_search_batch(idx, arr)
            assert np.array_equal(klp, np.array(case["exact_kl"])[sel]), (key, m)
        for z in (0, 1, 2):
            sel = [i for i, zz in enumerate(case["inexact_z"]) if zz == z]
            if not sel:
                continue
            ms = fm.inexact_search_batch(idx, [case["inexact_patterns"][i] for i in sel], z)
            grow = case["inexact_row"]
            for j, i in enumerate(sel):
                a, b = grow[i], grow[i + 1]
                want = [fm.MatchResult(fm.BwmInterval(k, l), d) for k, l, d in
                        zip(case["inexact_k"][a:b], case["inexact_l"][a:b], case["inexact_diffs"][a:b])]
                got = ms.results(j)
                assert got == want, (key, case["inexact_patterns"][i], z)
                hits, _ = fm.collect_hits(idx, got, len(case["inexact_patterns"][i]))
                assert [[h.global_pos, h.diffs] for h in hits] == case["hits"][i], key
        assert list(fm.locate_rows(idx, np.arange(n + 1))) == case["locate"], key
        sym, prev = fm.psi_inverse_batch(idx, np.arange(n + 1))
        got = [[-1, -1] if s == 255 else [int(s), int(p)] for s, p in zip(sym, prev)]
        assert got == case["psi"], key


def test_config0_exact_full(gpu):
    wl = workloads.config0()
    idx = fm.build_index(wl.text)
    want = np.load(GOLDEN / "config0_exact.npz")["kl"].astype(np.int64)
    kl, _ = fm.exact_search_batch(idx, wl.patterns)  # packed kernel
    assert np.array_equal(kl, want)
    kl2, _ = fm.exact_search_batch(idx, [codes_to_str(p) for p in wl.patterns[:2000]])  # general kernel
    assert np.array_equal(kl2, want[:2000])


def test_config1_occ_full(gpu):
    wl = workloads.config1()
    idx = fm.build_index(wl.text)
    got = fm.occ_pair_batch(idx, wl.pairs[:, 0], wl.pairs[:, 1])
    meta_path = GOLDEN / "config1_meta.json"
    if meta_path.exists():
        meta = json.loads(meta_path.read_text())
        assert hashlib.sha256(got.tobytes()).hexdigest() == meta["occ_sha256"]
    want = orc.occ_pair_batch(orc.OracleIndex(idx), wl.pairs[:, 0], wl.pairs[:, 1])
    assert np.array_equal(got, want)


def test_occ_device_tensor_path(gpu):
    import torch

    wl = workloads.config1(count=1 << 20)
    idx = fm.build_index(wl.text)
    kl = np.stack([wl.pairs[:, 0] + 1, wl.pairs[:, 1]], axis=1).astype(np.int32)
    d_out = fm.occ_pair_batch(idx, torch.from_numpy(kl).to(gpu))
    torch.cuda.synchronize()
    host = fm.occ_pair_batch(idx, wl.pairs[:, 0], wl.pairs[:, 1])
    assert np.array_equal(d_out.cpu().numpy().view(np.uint32), host)


def test_inexact_random_vs_oracle(gpu):
    rng = np.random.Generator(np.random.PCG64(4242))
    text = rng.integers(0, 4, 200_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    for m, z, count in ((5, 2, 300), (19, 1, 3000), (32, 1, 3000), (32, 0, 2000), (20, 2, 300),
                        (50, 1, 500), (80, 1, 300), (4, 3, 40), (6, 3, 60)):
        offs = rng.integers(0, text.size - m + 1, count)
        pats = workloads.substrings(text, offs, m)
        pats = workloads.mutate(pats.reshape(-1), 0.03, rng).reshape(count, m)
        pats[1::3] = rng.integers(0, 4, pats[1::3].shape, dtype=np.uint8)
        ms = fm.inexact_search_batch(idx, pats, z)
        row, k, l, d, steps = orc.inexact_batch(ox, pats, z)
        assert np.array_equal(ms.offsets, row), (m, z)
        assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
        assert np.array_equal(ms.diffs, d), (m, z)
        if z == 1 and m >= 19:  # no result-buffer retries here: pruned work <= DFS + bound pass
            assert ms.steps <= steps + count * m, (m, z, ms.steps, steps)


def test_exact_edge_cases(gpu):
    rng = np.random.Generator(np.random.PCG64(99))
    text = rng.integers(0, 4, 50_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    pats = []
    for m in (1, 2, 31, 32, 33, 64, 65, 100, 150):
        for _ in range(20):
            s = int(rng.integers(0, text.size - m + 1))
            pats.append(codes_to_str(text[s:s + m]))
            pats.append(codes_to_str(rng.integers(0, 4, m, dtype=np.uint8)))
    kl, _ = fm.exact_search_batch(idx, pats)
    assert np.array_equal(kl, orc.exact_batch(ox, pats))
    kl, deg = fm.exact_search_batch(idx, ["acgt", "ACNT", "A"])
    assert deg.tolist() == [False, True, False] and tuple(kl[1]) == (1, 0)
    assert tuple(kl[0]) == tuple(orc.exact_batch(ox, ["ACGT"])[0])


def test_config2_subsample_vs_oracle(gpu):
    wl = workloads.config2(n_reads=20_000)
    idx = fm.build_index(wl.text)
    ms = fm.inexact_search_batch(idx, wl.patterns, 1)
    row, k, l, d, _ = orc.inexact_batch(orc.OracleIndex(idx), wl.patterns, 1)
    assert np.array_equal(ms.offsets, row)
    assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
    assert np.array_equal(ms.diffs, d)


@pytest.mark.parametrize("words", [6, 14])
def test_alternate_line_layouts(small_cases, gpu, words, monkeypatch):
    """The W=6 (64 B) and W=14 (128 B) line layouts give identical results."""
    monkeypatch.setenv("FMG_LINE_WORDS", str(words))
    for key in ("1000_15", "2500_16", "129_11", "4_2"):
        case = small_cases[key]
        n = case["n"]
        idx = fm.build_index(small_text(n, case["seed"]))
        occ = fm.occ_pair_batch(idx, case["occ_low"], case["occ_high"])
        assert np.array_equal(occ.astype(np.int64), np.array(case["occ"])), key
        kl, _ = fm.exact_search_batch(idx, case["exact_patterns"])
        assert np.array_equal(kl, np.array(case["exact_kl"])), key
        assert list(fm.locate_rows(idx, np.arange(n + 1))) == case["locate"], key
        sel = [i for i, zz in enumerate(case["inexact_z"]) if zz == 1]
        ms = fm.inexact_search_batch(idx, [case["inexact_patterns"][i] for i in sel], 1)
        for j, i in enumerate(sel):
            a, b = case["inexact_row"][i], case["inexact_row"][i + 1]
            assert [(r.interval.k, r.interval.l, r.diffs_used) for r in ms.results(j)] == list(
                zip(case["inexact_k"][a:b], case["inexact_l"][a:b], case["inexact_diffs"][a:b])), key
    wl = workloads.config1(count=1 << 20)
    idx = fm.build_index(wl.text)
    got = fm.occ_pair_batch(idx, wl.pairs[:, 0], wl.pairs[:, 1])
    want = orc.occ_pair_batch(orc.OracleIndex(idx), wl.pairs[:, 0], wl.pairs[:, 1])
    assert np.array_equal(got, want)
    pats = workloads.substrings(wl.text, np.arange(0, 1 << 20, 97)[:5000], 24)
    kl, _ = fm.exact_search_batch(idx, pats)
    assert np.array_equal(kl, orc.exact_batch(orc.OracleIndex(idx), pats))


def test_config3_small_scale_vs_oracle(gpu, monkeypatch):
    """Config-3 generator at 1/150 scale: exact and z=1 on packed 19-bp seeds, through the
    packed host entry point, one-directional (no reverse index) and then bidirectional in its
    flat (the config-3 default at scale: one warp per pattern over its one-edit neighbourhood,
    gathers into the level-(K+1) table), split (edit range split at 3m/4, case-A jumps into the
    level-(K+1) table), level-synchronous and per-thread forms."""
    import ctypes as ct

    from paper_1811_06127_b200 import _lib

    wl = workloads.config3(n_reads=3000, n=20_000_000)
    idx = fm.build_index(wl.text)
    seeds = workloads.unpack_patterns(wl.packed, 19)
    ox = orc.OracleIndex(idx)
    kl, _ = fm.exact_search_batch(idx, seeds)  # builds the level-(K+1) k-mer table too
    assert np.array_equal(kl, orc.exact_batch(ox, seeds))
    orow, ok, ol, od, _ = orc.inexact_batch(ox, seeds, 1)
    lib = _lib.load()
    dix = idx.device_index()
    for engine in (None, "flat", "split", "sync", "dfs"):
        if engine is not None:
            if engine != "flat":
                dix.ensure_reverse()
            monkeypatch.setenv("FMG_BIDIR_ENGINE", engine)
        h = ct.c_void_p()
        _lib.check(lib.fmg_inexact_packed_host(dix.handle, wl.packed.ctypes.data, 19, wl.packed.size, 1, ct.byref(h)))
        tot = ct.c_uint64()
        lib.fmg_matches_size(h, ct.byref(tot), None)
        row = np.empty(wl.packed.size + 1, np.uint64)
        k = np.empty(tot.value, np.uint32)
        l = np.empty(tot.value, np.uint32)
        d = np.empty(tot.value, np.uint8)
        lib.fmg_matches_copy(h, row.ctypes.data, k.ctypes.data, l.ctypes.data, d.ctypes.data, 1)
        lib.fmg_matches_free(h)
        assert np.array_equal(row, orow) and np.array_equal(k.astype(np.int64), ok), engine
        assert np.array_equal(l.astype(np.int64), ol) and np.array_equal(d, od), engine


def test_config1h_sample_vs_oracle(gpu):
    """Config 1-H (1 Gbp, HBM-resident index): 2^20 pairs of the bench workload."""
    wl = workloads.config1h(count=1 << 20)
    idx = fm.build_index(wl.text, builder="gpu")
    got = fm.occ_pair_batch(idx, wl.pairs[:, 0], wl.pairs[:, 1])
    want = orc.occ_pair_batch(orc.OracleIndex(idx), wl.pairs[:, 0], wl.pairs[:, 1])
    assert np.array_equal(got, want)
    idx.release_device()


@pytest.mark.slow
def test_config2_full_vs_oracle(gpu):
    """All 1,000,000 config-2 seeds, z = 1, every result bit-exact."""
    wl = workloads.config2()
    idx = fm.build_index(wl.text)
    ms = fm.inexact_search_batch(idx, wl.patterns, 1)
    row, k, l, d, _ = orc.inexact_batch(orc.OracleIndex(idx), wl.patterns, 1)
    assert np.array_equal(ms.offsets, row)
    assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
    assert np.array_equal(ms.diffs, d)


def test_config4_first_chunk_vs_oracle(gpu):
    """The first 2^22 seeds of config 4 (identical to the full set's first chunk)."""
    wl = workloads.config4(count=1 << 22)
    idx = fm.build_index(wl.text, builder="gpu")
    seeds = workloads.unpack_patterns(wl.packed, 20)
    kl, _ = fm.exact_search_batch(idx, seeds)
    ox = orc.OracleIndex(idx)
    assert np.array_equal(kl[: 1 << 20], orc.exact_batch(ox, seeds[: 1 << 20]))
    hit = kl[:, 0] <= kl[:, 1]
    assert abs(hit.mean() - 0.8) < 0.01  # 80% exact substrings, random 20-mers ~never occur
    idx.release_device()


def test_z1_engines_agree(gpu, monkeypatch):
    """z = 1 on an L2-resident repeat genome: the bidirectional engine (default once a
    reverse index is attached) in its level-synchronous (default here), split and per-thread
    forms, the one-directional level-synchronous engine and the DFS engine give identical
    result sets, equal to the oracle's."""
    wl = workloads.config2(n_reads=20_000, n=8_000_000)
    idx = fm.build_index(wl.text)
    a = fm.inexact_search_batch(idx, wl.patterns, 1)  # >= BIDIR_MIN_N: bidirectional, sync form
    assert idx.device_index()._has_reverse
    for eng in ("split", "dfs"):
        monkeypatch.setenv("FMG_BIDIR_ENGINE", eng)
        x = fm.inexact_search_batch(idx, wl.patterns, 1)
        assert np.array_equal(a.offsets, x.offsets) and np.array_equal(a.k, x.k), eng
        assert np.array_equal(a.l, x.l) and np.array_equal(a.diffs, x.diffs), eng
    monkeypatch.delenv("FMG_BIDIR_ENGINE")
    monkeypatch.setenv("FMG_INEXACT_BIDIR", "0")
    c = fm.inexact_search_batch(idx, wl.patterns, 1)  # level-synchronous z1 engine
    monkeypatch.setenv("FMG_INEXACT_DFS", "1")
    b = fm.inexact_search_batch(idx, wl.patterns, 1)  # one-directional DFS
    for x in (b, c):
        assert np.array_equal(a.offsets, x.offsets) and np.array_equal(a.k, x.k)
        assert np.array_equal(a.l, x.l) and np.array_equal(a.diffs, x.diffs)
    row, k, l, d, _ = orc.inexact_batch(orc.OracleIndex(idx), wl.patterns, 1)
    assert np.array_equal(a.offsets, row) and np.array_equal(a.k.astype(np.int64), k)
    assert np.array_equal(a.l.astype(np.int64), l) and np.array_equal(a.diffs, d)


def test_exact_kmer_table_paths(gpu):
    """>= 1024 patterns use the tables: here prefix levels 1..9 and the exact-search level 12
    (floor(log4 n) + 4).  Lengths below 9 (one prefix-level gather is the answer), 9..11
    (level 9 + steps), at and above 12 (level 12 + steps), present and absent, packed and CSR
    inputs — all identical to the oracle."""
    rng = np.random.Generator(np.random.PCG64(606))
    text = rng.integers(0, 4, 200_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    pats = []
    for _ in range(40_000):
        m = int(rng.integers(1, 41))
        if rng.random() < 0.6:
            s = int(rng.integers(0, text.size - m + 1))
            pats.append(codes_to_str(text[s:s + m]))
        else:
            pats.append(codes_to_str(rng.integers(0, 4, m, dtype=np.uint8)))
    kl, _ = fm.exact_search_batch(idx, pats)  # CSR kernel
    assert np.array_equal(kl, orc.exact_batch(ox, pats))
    for m in (5, 8, 9, 10, 20):
        arr = rng.integers(0, 4, (1 << 15, m), dtype=np.uint8)
        arr[::2] = workloads.substrings(text, rng.integers(0, text.size - m + 1, arr[::2].shape[0]), m)
        klp, _ = fm.exact_search_batch(idx, arr)  # packed kernel
        assert np.array_equal(klp, orc.exact_batch(ox, arr)), m


def _scale_cases():
    path = GOLDEN / "scale_cases.json"
    assert path.exists(), "tests/golden/scale_cases.json missing (make_golden.py scale)"
    return json.loads(path.read_text())


def test_scale_golden_config4_config1h(gpu):
    """Reference outputs (fmpm run on this text, tests/golden/make_golden.py scale) on the
    1 Gbp config-4 / 1-H text, GPU-built index: the first 16k config-4 seeds (exact) and
    the first 4k config-1-H Occ pairs."""
    cases = _scale_cases()
    wl4 = workloads.config4(count=1 << 14)
    idx = fm.build_index(wl4.text, builder="gpu")
    seeds = workloads.unpack_patterns(wl4.packed, 20)
    kl, _ = fm.exact_search_batch(idx, seeds)  # 16k >= 1024: k-mer table path
    assert np.array_equal(kl.astype(np.int64), np.array(cases["config4_first16k_kl"], dtype=np.int64))
    wl1h = workloads.config1h(count=1 << 12)
    got = fm.occ_pair_batch(idx, wl1h.pairs[:, 0], wl1h.pairs[:, 1])
    assert np.array_equal(got.astype(np.int64), np.array(cases["config1h_first4k_occ"], dtype=np.int64))
    idx.release_device()


def test_scale_golden_config2(gpu):
    """Reference z = 1 result lists for the first 2000 config-2 seeds (1M-read workload)."""
    cases = _scale_cases()["config2_first2k_z1"]
    wl = workloads.config2()
    idx = fm.build_index(wl.text)
    ms = fm.inexact_search_batch(idx, wl.patterns[:2000], 1)
    off = ms.offsets.astype(np.int64)
    for q, want in enumerate(cases):
        a, b = off[q], off[q + 1]
        got = list(zip(ms.k[a:b].tolist(), ms.l[a:b].tolist(), ms.diffs[a:b].tolist()))
        assert got == [tuple(x) for x in want], q


@pytest.mark.parametrize("z,lens", [(1, (1, 2, 3, 8, 9, 10, 19, 32, 40)), (2, (1, 2, 5, 9, 10, 20)), (3, (1, 3, 6, 9, 10)),
                                    (1, (70, 90))])
def test_inexact_prefix_table_paths(gpu, monkeypatch, z, lens):
    """The DFS engine with the prefix table (>= 1024 patterns; K = 9 here): shallow nodes
    stepped through the table, the depth-K hand-over to index lines, length-1..3 patterns
    whose results come from shallow nodes (root skip), long (> 64) patterns — identical to
    the oracle and to the table-less engine."""
    monkeypatch.setenv("FMG_INEXACT_DFS", "1")
    rng = np.random.Generator(np.random.PCG64(777 + z))
    text = rng.integers(0, 4, 200_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    pats = []
    for _ in range(1200):
        m = int(rng.choice(lens))
        if rng.random() < 0.6:
            s = int(rng.integers(0, text.size - m + 1))
            p = text[s:s + m].copy()
            if m > 4 and rng.random() < 0.5:
                p[int(rng.integers(0, m))] = rng.integers(0, 4)
        else:
            p = rng.integers(0, 4, m, dtype=np.uint8)
        pats.append(codes_to_str(p))
    ms = fm.inexact_search_batch(idx, pats, z)
    row, k, l, d, _ = orc.inexact_batch(ox, pats, z)
    assert np.array_equal(ms.offsets, row)
    assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
    assert np.array_equal(ms.diffs, d)
    monkeypatch.setenv("FMG_INEXACT_LUT", "0")
    b = fm.inexact_search_batch(idx, pats, z)
    assert np.array_equal(b.offsets, ms.offsets) and np.array_equal(b.k, ms.k) and np.array_equal(b.diffs, ms.diffs)


@pytest.mark.parametrize("engine", ["split", "sync", "dfs"])
@pytest.mark.parametrize("n,lens", [(200_000, (1, 2, 3, 5, 8, 9, 10, 11, 19, 20, 32, 33, 47, 64)),
                                    (3_000, (1, 2, 4, 7, 12, 19, 25)), (40, (1, 2, 3, 6, 9, 14))])
def test_inexact_bidirectional_engine(gpu, monkeypatch, n, lens, engine):
    """z = 1 through the bidirectional engine (reverse index attached, both prefix tables):
    patterns cut from anywhere (incl. the text's very start and end, which exercises the
    forward extension's '$' term), mutated or random, lengths 1..64 — identical to the
    oracle and to the one-directional DFS engine."""
    monkeypatch.setenv("FMG_BIDIR_MIN_N", "0")
    monkeypatch.setenv("FMG_INEXACT_DFS", "1")
    monkeypatch.setenv("FMG_BIDIR_ENGINE", engine)
    rng = np.random.Generator(np.random.PCG64(31337 + n))
    text = rng.integers(0, 4, n, dtype=np.uint8)
    idx = fm.build_index(text)
    pats = []
    for r in range(3000):
        m = int(rng.choice(lens))
        if m > n:
            m = n
        kind = r % 5
        if kind == 0:  # a suffix of the text
            p = text[n - m:].copy()
        elif kind == 1:  # a prefix of the text
            p = text[:m].copy()
        elif kind == 2:
            p = rng.integers(0, 4, m, dtype=np.uint8)
        else:
            s = int(rng.integers(0, n - m + 1))
            p = text[s:s + m].copy()
        if m > 2 and rng.random() < 0.5:  # one random edit
            j = int(rng.integers(0, m))
            e = rng.random()
            if e < 0.4:
                p[j] = (p[j] + 1 + rng.integers(0, 3)) % 4
            elif e < 0.7:
                p = np.delete(p, j)
            else:
                p = np.insert(p, j, rng.integers(0, 4))
        pats.append(codes_to_str(p[:64]))
    ms = fm.inexact_search_batch(idx, pats, 1)
    assert idx.device_index()._has_reverse
    ox = orc.OracleIndex(idx)
    row, k, l, d, _ = orc.inexact_batch(ox, pats, 1)
    assert np.array_equal(ms.offsets, row)
    assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
    assert np.array_equal(ms.diffs, d)
    monkeypatch.setenv("FMG_INEXACT_BIDIR", "0")
    b = fm.inexact_search_batch(idx, pats, 1)
    assert np.array_equal(b.offsets, ms.offsets) and np.array_equal(b.k, ms.k) and np.array_equal(b.diffs, ms.diffs)
    assert ms.steps < b.steps  # the point of the engine


@pytest.mark.parametrize("n,lens", [(200_000, (1, 2, 3, 5, 8, 9, 10, 11, 12, 19, 20, 27, 31)),
                                    (3_000, (1, 2, 4, 7, 12, 19, 25, 31)), (40, (1, 2, 3, 6, 9, 14)),
                                    (200_000, (9, 10, 11)), (200_000, (17, 18, 19))])
@pytest.mark.parametrize("filt", ["default", "off", "copies1_d1", "copies2_d3", "overflow"])
def test_inexact_flat_engine(gpu, monkeypatch, n, lens, filt):
    """z = 1 through the flat engine (kernels_flat.cuh: a warp per pattern, one table gather
    per string of the one-edit neighbourhood, survivors extended level by level): patterns
    of mixed lengths 1..31 cut from anywhere (text start / end included), mutated or random,
    repeats — identical to the oracle; every NR instantiation (m <= 11, <= 19, <= 31); with
    the presence filter in its default shape (B = table level + 2, one copy per four window
    positions), off, and in two other shapes (one ungrouped copy of level + 1; two copies of
    level + 3)."""
    monkeypatch.setenv("FMG_BIDIR_ENGINE", "flat")
    if filt == "off":
        monkeypatch.setenv("FMG_FLAT_FILTER", "0")
    elif filt == "overflow":  # a survivor queue of 3 entries per pattern: most patterns go to the retry passes
        monkeypatch.setenv("FMG_FLAT_PER_PAT", "3")
    elif filt != "default":
        copies, d = filt.split("_")
        monkeypatch.setenv("FMG_FLAT_FILTER_NO", copies[-1])
        monkeypatch.setenv("FMG_FLAT_FILTER_D", d[-1])
    rng = np.random.Generator(np.random.PCG64(99 + n + len(lens)))
    text = rng.integers(0, 4, n, dtype=np.uint8)
    if n >= 3000:  # a tandem repeat and a homopolymer run: many candidates occur, many spell the same string
        text[1000:1400] = np.tile(text[1000:1010], 40)
        text[2000:2100] = 2
    idx = fm.build_index(text)
    pats = []
    for r in range(3000):
        m = min(int(rng.choice(lens)), n)
        kind = r % 6
        if kind == 0:
            p = text[n - m:].copy()
        elif kind == 1:
            p = text[:m].copy()
        elif kind == 2:
            p = rng.integers(0, 4, m, dtype=np.uint8)
        elif kind == 3 and n >= 3000:
            s = int(rng.integers(990, 2100 - m))
            p = text[s:s + m].copy()
        else:
            s = int(rng.integers(0, n - m + 1))
            p = text[s:s + m].copy()
        if m > 2 and rng.random() < 0.5:  # one random edit
            j = int(rng.integers(0, m))
            e = rng.random()
            if e < 0.4:
                p[j] = (p[j] + 1 + rng.integers(0, 3)) % 4
            elif e < 0.7:
                p = np.delete(p, j)
            else:
                p = np.insert(p, j, rng.integers(0, 4))
        pats.append(codes_to_str(p[:31]))
    ms = fm.inexact_search_batch(idx, pats, 1)
    row, k, l, d, _ = orc.inexact_batch(orc.OracleIndex(idx), pats, 1)
    assert np.array_equal(ms.offsets, row)
    assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l)
    assert np.array_equal(ms.diffs, d)
    # the filter really was in play (or really was not)
    import ctypes as ct

    from paper_1811_06127_b200 import _lib

    fb, fg, fc = ct.c_uint32(), ct.c_uint32(), ct.c_uint32()
    _lib.check(_lib.load().fmgx_flat_filter_info(idx.device_index().handle, ct.byref(fb), ct.byref(fg),
                                                 ct.byref(fc), None))
    kk, nb = ct.c_uint32(), ct.c_uint64()
    _lib.check(_lib.load().fmgx_prefix_table(idx.device_index().handle, ct.byref(kk), ct.byref(nb)))
    depth = 2 if filt in ("default", "overflow") else int(filt[-1]) if filt != "off" else 0
    if filt == "off":
        assert fc.value == 0
    elif max(lens) >= kk.value + depth:  # some candidate is long enough for a window
        assert fb.value == kk.value + depth and fg.value * fc.value >= fb.value
        assert fc.value == ((fb.value + 3) // 4 if filt in ("default", "overflow") else int(filt[6]))
    monkeypatch.setenv("FMG_BIDIR_ENGINE", "dfs")
    b = fm.inexact_search_batch(idx, pats, 1)
    assert np.array_equal(b.offsets, ms.offsets) and np.array_equal(b.k, ms.k) and np.array_equal(b.diffs, ms.diffs)


def test_exact_packed_host_pinned_and_pageable(gpu):
    """fmg_exact_packed_host with pinned buffers (small batch: the kernel reads and writes the host
    mappings directly) and with pageable ones (staged pipeline): both equal the oracle."""
    import ctypes as ct

    import torch

    from paper_1811_06127_b200 import _lib, pack_patterns_u64

    wl = workloads.config0()
    idx = fm.build_index(wl.text)
    want = orc.exact_batch(orc.OracleIndex(idx), wl.patterns)
    packed = pack_patterns_u64(wl.patterns)
    lib, dix = _lib.load(), idx.device_index()
    out = np.empty((packed.size, 2), dtype=np.uint32)  # pageable in, pageable out
    _lib.check(lib.fmg_exact_packed_host(dix.handle, packed.ctypes.data, 32, packed.size, out.ctypes.data))
    assert np.array_equal(out, want)
    pin_in = torch.from_numpy(packed.view(np.int64)).pin_memory()
    pin_out = torch.zeros((packed.size, 2), dtype=torch.int32).pin_memory()
    for _ in range(3):
        pin_out.zero_()
        _lib.check(lib.fmg_exact_packed_host(dix.handle, pin_in.data_ptr(), 32, packed.size, pin_out.data_ptr()))
        assert np.array_equal(pin_out.numpy().view(np.uint32), want)
    # pinned in, pageable out: staged
    out2 = np.empty_like(out)
    _lib.check(lib.fmg_exact_packed_host(dix.handle, pin_in.data_ptr(), 32, packed.size, out2.ctypes.data))
    assert np.array_equal(out2, want)


def test_wants_reverse_follows_the_engine_choice(gpu, monkeypatch):
    """fmg_inexact_wants_reverse: 1 only when a bidirectional z = 1 engine would take the batch;
    the Python layer then skips the reverse index for the flat engine."""
    rng = np.random.Generator(np.random.PCG64(5))
    text = rng.integers(0, 4, 1 << 22, dtype=np.uint8)
    idx = fm.build_index(text)
    dix = idx.device_index()
    assert dix.wants_reverse(4096, 19, 1)          # L2-resident lines: the bidirectional engines
    assert not dix.wants_reverse(4096, 19, 2)      # z != 1: the DFS engine
    assert not dix.wants_reverse(100, 19, 1)       # small batch
    monkeypatch.setenv("FMG_BIDIR_ENGINE", "flat")
    assert not dix.wants_reverse(4096, 19, 1)      # the flat engine reads none
    pats = [codes_to_str(text[s:s + 19]) for s in rng.integers(0, text.size - 19, 2048)]
    ms = fm.inexact_search_batch(idx, pats, 1)
    assert not dix._has_reverse
    row, k, l, d, _ = orc.inexact_batch(orc.OracleIndex(idx), pats, 1)
    assert np.array_equal(ms.offsets, row) and np.array_equal(ms.k.astype(np.int64), k)
    assert np.array_equal(ms.l.astype(np.int64), l) and np.array_equal(ms.diffs, d)
    monkeypatch.setenv("FMG_BIDIR_ENGINE", "split")
    assert dix.wants_reverse(4096, 19, 1)


def test_inexact_repeated_calls_reuse_dedup_table(gpu, monkeypatch):
    """The dedup hash table persists in the index between calls (epoch-tagged, zeroed only on
    allocation): back-to-back calls with different batches, budgets and engines on one index
    must each equal the oracle — stale entries of earlier calls never read as results."""
    monkeypatch.setenv("FMG_BIDIR_MIN_N", "0")
    rng = np.random.Generator(np.random.PCG64(4242))
    text = rng.integers(0, 4, 300_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    for call, (z, n_pat, m, env) in enumerate([(1, 3000, 20, None), (1, 1500, 24, None), (2, 1200, 16, None),
                                               (1, 3000, 20, "FMG_INEXACT_BIDIR"), (1, 2000, 18, None)]):
        if env:
            monkeypatch.setenv(env, "0")
        pats = workloads.substrings(text, rng.integers(0, text.size - m + 1, n_pat), m).copy()
        mut = rng.random(n_pat) < 0.5
        pos = rng.integers(0, m, n_pat)
        pats[mut, pos[mut]] = (pats[mut, pos[mut]] + 1) % 4
        ms = fm.inexact_search_batch(idx, pats, z)
        row, k, l, d, _ = orc.inexact_batch(ox, pats, z)
        assert np.array_equal(ms.offsets, row), call
        assert np.array_equal(ms.k.astype(np.int64), k) and np.array_equal(ms.l.astype(np.int64), l), call
        assert np.array_equal(ms.diffs, d), call
        if env:
            monkeypatch.delenv(env)


def test_device_pattern_validation_errors(gpu):
    """Device-side pattern checks of the C ABI (k_check_patterns): a code > 3, an empty
    pattern and offsets not starting at 0 are EINVAL with the reference's messages, at any
    position in a large batch and from an unaligned codes pointer; a valid call still works."""
    import ctypes as ct

    import torch

    from paper_1811_06127_b200 import _lib

    lib = _lib.load()
    rng = np.random.Generator(np.random.PCG64(99))
    text = rng.integers(0, 4, 50_000, dtype=np.uint8)
    idx = fm.build_index(text)
    dix = idx.device_index()
    n, m = 100_000, 12
    base = workloads.substrings(text, rng.integers(0, text.size - m + 1, n), m).reshape(-1)

    def run(codes: np.ndarray, offs: np.ndarray, shift: int = 0, z: int = 1):
        buf = torch.zeros(codes.size + 8, dtype=torch.uint8, device=gpu)
        buf[shift:shift + codes.size] = torch.from_numpy(codes).to(gpu)
        d_off = torch.from_numpy(offs.astype(np.int64)).to(gpu)
        h = ct.c_void_p()
        rc = lib.fmg_inexact(dix.handle, buf.data_ptr() + shift, d_off.data_ptr(), offs.size - 1, z, ct.byref(h), None)
        if rc == 0:
            lib.fmg_matches_free(h)
        return rc, _lib.last_error()

    offs = np.arange(0, (n + 1) * m, m, dtype=np.uint64)
    for shift in (0, 1, 3):
        assert run(base, offs, shift)[0] == 0
        for pos in (0, 7, base.size // 2 + 5, base.size - 1):
            bad = base.copy()
            bad[pos] = 4 + pos % 200
            rc, msg = run(bad, offs, shift)
            assert rc == 1 and "symbol code" in msg, (shift, pos, rc, msg)
    empty = offs.copy()
    empty[n // 3 + 1] = empty[n // 3]  # pattern n//3 empty (and the next one twice as long)
    rc, msg = run(base, empty)
    assert rc == 1 and "empty" in msg, msg
    rc, msg = run(base[m:], offs[1:] - offs[1] + m)  # offsets[0] = m != 0
    assert rc == 1 and "start at 0" in msg, msg
    ms = fm.inexact_search_batch(idx, base.reshape(n, m)[:2000], 1)  # still healthy
    row, k, _, _, _ = orc.inexact_batch(orc.OracleIndex(idx), base.reshape(n, m)[:2000], 1)
    assert np.array_equal(ms.offsets, row) and np.array_equal(ms.k.astype(np.int64), k)


def test_concurrent_host_calls_one_index(gpu, monkeypatch):
    """Four host threads search one index at once (exact and z = 1, host entry points on each
    thread's own streams; the dedup-table lease falls back to per-call tables for the threads
    that find it taken): every result equals the oracle's."""
    import threading

    monkeypatch.setenv("FMG_BIDIR_MIN_N", "0")
    rng = np.random.Generator(np.random.PCG64(2024))
    text = rng.integers(0, 4, 400_000, dtype=np.uint8)
    idx = fm.build_index(text)
    ox = orc.OracleIndex(idx)
    batches = []
    for t in range(4):
        m = 18 + t
        pats = workloads.substrings(text, rng.integers(0, text.size - m + 1, 4000), m).copy()
        pats[::3, m // 2] = (pats[::3, m // 2] + 1) % 4
        batches.append(pats)
    fm.exact_search_batch(idx, batches[0])  # build the tables once before the threads race
    fm.inexact_search_batch(idx, batches[0], 1)
    out = [None] * 4
    errors = []

    def work(t):
        try:
            kl, _ = fm.exact_search_batch(idx, batches[t])
            ms = fm.inexact_search_batch(idx, batches[t], 1)
            out[t] = (kl, ms)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t in range(4):
        kl, ms = out[t]
        assert np.array_equal(kl, orc.exact_batch(ox, batches[t])), t
        row, k, l, d, _ = orc.inexact_batch(ox, batches[t], 1)
        assert np.array_equal(ms.offsets, row) and np.array_equal(ms.k.astype(np.int64), k), t
        assert np.array_equal(ms.l.astype(np.int64), l) and np.array_equal(ms.diffs, d), t
