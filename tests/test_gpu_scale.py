"""Parity at BASELINE scale: config 3 at its full 3.1 Gbp (the only config whose
rows exceed 2^31) through every z = 1 engine form, and hit lists (collect_hits,
search.py:211-267) on configs 0, 2, 3 and 4 — against the oracle on large
deterministic subsamples and against the reference's own outputs
(tests/golden/scale3_cases.json, hits_cases.json, from make_golden.py)."""

import ctypes as ct
import json

import numpy as np
import pytest

import paper_1811_06127_b200 as fm
from conftest import GOLDEN
from oracle import oracle as orc
from paper_1811_06127_b200 import _lib, workloads

pytestmark = pytest.mark.gpu

C3_READS = 8192  # tests/golden/make_golden.py C3_READS: 114,688 seeds


def _hits(idx, kl_or_ms, m, n_pat):
    """Our hit lists, per pattern, as [(pos, diffs)]."""
    if isinstance(kl_or_ms, np.ndarray):
        pid, k, l, d = np.arange(n_pat), kl_or_ms[:, 0], kl_or_ms[:, 1], np.zeros(n_pat)
    else:
        cnt = np.diff(kl_or_ms.offsets.astype(np.int64))
        pid, k, l, d = np.repeat(np.arange(n_pat), cnt), kl_or_ms.k, kl_or_ms.l, kl_or_ms.diffs
    hp, pos, hd, _, _, _ = fm.collect_hits_batch(idx, pid, k, l, d, np.full(n_pat, m))
    return hp, pos, hd


def _oracle_hits(ox, kl_or_csr, m, n_pat):
    if isinstance(kl_or_csr, np.ndarray):
        return orc.collect_hits(ox, np.arange(n_pat), kl_or_csr[:, 0], kl_or_csr[:, 1], np.zeros(n_pat),
                                np.full(n_pat, m))
    row, k, l, d = kl_or_csr
    cnt = np.diff(row.astype(np.int64))
    return orc.collect_hits(ox, np.repeat(np.arange(n_pat), cnt), k, l, d, np.full(n_pat, m))


def _per_pattern(hp, pos, hd, n_pat):
    out = [[] for _ in range(n_pat)]
    for p, x, d in zip(hp.tolist(), pos.tolist(), hd.tolist()):
        if p < n_pat:
            out[p].append((x, d))
    return out


def _same(a, b):
    return all(np.array_equal(np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64)) for x, y in zip(a, b))


def _inexact_packed(lib, dix, packed, m):
    h = ct.c_void_p()
    _lib.check(lib.fmg_inexact_packed_host(dix.handle, packed.ctypes.data, m, packed.size, 1, ct.byref(h)))
    try:
        tot = ct.c_uint64()
        lib.fmg_matches_size(h, ct.byref(tot), None)
        row = np.empty(packed.size + 1, np.uint64)
        k = np.empty(tot.value, np.uint32)
        l = np.empty(tot.value, np.uint32)
        d = np.empty(tot.value, np.uint8)
        _lib.check(lib.fmg_matches_copy(h, row.ctypes.data, k.ctypes.data, l.ctypes.data, d.ctypes.data, 1))
    finally:
        lib.fmg_matches_free(h)
    return row, k, l, d


@pytest.fixture(scope="module")
def c3():
    wl = workloads.config3(n_reads=C3_READS)
    idx = fm.build_index(wl.text, builder="gpu")
    yield wl, idx
    idx.release_device()


def test_config3_full_scale_exact_and_hits(gpu, c3):
    wl, idx = c3
    gold = json.loads((GOLDEN / "scale3_cases.json").read_text())
    assert gold["n"] == idx.n == 3_100_000_000
    seeds = workloads.unpack_patterns(wl.packed, 19)
    kl, _ = fm.exact_search_batch(idx, seeds)
    ox = orc.OracleIndex(idx)
    assert np.array_equal(kl, orc.exact_batch(ox, seeds))                     # all 114,688 seeds
    assert np.array_equal(kl[:2048], np.array(gold["exact"], dtype=np.int64))  # the reference itself
    assert (kl[:, 0] > (1 << 31)).any() and (kl[:, 1] < kl[:, 0]).any()      # rows past 2^31, misses
    ours = _hits(idx, kl, 19, seeds.shape[0])
    want = _oracle_hits(ox, kl, 19, seeds.shape[0])
    assert all(np.array_equal(a, b) for a, b in zip(ours, want))
    per = _per_pattern(*ours, 2048)
    checked = 0
    for got, ref in zip(per, gold["exact_hits"]):
        if ref is not None:
            assert [tuple(x) for x in ref] == got
            checked += 1
    assert checked > 1500


# engines that read the reverse index first: its GPU build wants ~36 bytes per character (112 GB
# here), which no longer fits once the flat engine's presence filter (43 GB) is resident
@pytest.mark.parametrize("engine", ["split", "sync", "dfs", "default", "onedir"])
def test_config3_full_scale_z1_every_engine(gpu, c3, monkeypatch, engine):
    wl, idx = c3
    gold = json.loads((GOLDEN / "scale3_cases.json").read_text())
    lib = _lib.load()
    dix = idx.device_index()
    if engine in ("split", "sync", "dfs"):
        dix.ensure_reverse()
        monkeypatch.setenv("FMG_BIDIR_ENGINE", engine)
    if engine == "onedir":
        monkeypatch.setenv("FMG_INEXACT_BIDIR", "0")
    # the default (flat) form on every seed; the other forms on the first 2^15
    count = wl.packed.size if engine == "default" else 1 << 15
    packed = np.ascontiguousarray(wl.packed[:count])
    seeds = workloads.unpack_patterns(packed, 19)
    row, k, l, d = _inexact_packed(lib, dix, packed, 19)
    ox = orc.OracleIndex(idx)
    orow, ok, ol, od, _ = orc.inexact_batch(ox, seeds, 1)
    assert np.array_equal(row, orow) and np.array_equal(k.astype(np.int64), ok)
    assert np.array_equal(l.astype(np.int64), ol) and np.array_equal(d, od)
    assert (k.astype(np.int64) > (1 << 31)).any()
    ref = [[tuple(x) for x in r] for r in gold["z1"]]
    for i in range(2048):
        a, b = int(row[i]), int(row[i + 1])
        assert list(zip(k[a:b].tolist(), l[a:b].tolist(), d[a:b].tolist())) == ref[i], i
    if engine == "default":
        ms = fm.MatchSet(row, k, l, d, 0)
        ours = _hits(idx, ms, 19, count)
        want = _oracle_hits(ox, (row, k, l, d), 19, count)
        assert all(np.array_equal(a, b) for a, b in zip(ours, want))
        per = _per_pattern(*ours, 2048)
        for got, r in zip(per, gold["z1_hits"]):
            if r is not None:
                assert [tuple(x) for x in r] == got


def test_hits_config0_config2_config4(gpu):
    gold = json.loads((GOLDEN / "hits_cases.json").read_text())
    # config 0: every pattern's exact hits vs the oracle, the first 1,000 vs the reference
    wl = workloads.config0()
    idx = fm.build_index(wl.text)
    ox = orc.OracleIndex(idx)
    kl, _ = fm.exact_search_batch(idx, wl.patterns)
    ours = _hits(idx, kl, 32, kl.shape[0])
    assert all(np.array_equal(a, b) for a, b in zip(ours, _oracle_hits(ox, kl, 32, kl.shape[0])))
    for got, ref in zip(_per_pattern(*ours, 1000), gold["config0_first1k_exact_hits"]):
        assert ref is None or [tuple(x) for x in ref] == got
    # config 2: z = 1 hits of the first 2^16 seeds vs the oracle, the first 500 vs the reference
    wl = workloads.config2()
    idx = fm.build_index(wl.text)
    ox = orc.OracleIndex(idx)
    pats = wl.patterns[: 1 << 16]
    ms = fm.inexact_search_batch(idx, pats, 1)
    ours = _hits(idx, ms, 32, pats.shape[0])
    orow, ok, ol, od, _ = orc.inexact_batch(ox, pats, 1)
    assert all(np.array_equal(a, b) for a, b in zip(ours, _oracle_hits(ox, (orow, ok, ol, od), 32, pats.shape[0])))
    for got, ref in zip(_per_pattern(*ours, 500), gold["config2_first500_z1_hits"]):
        assert ref is None or [tuple(x) for x in ref] == got
    idx.release_device()
    # config 4 (1 Gbp): exact hits of the first 2^16 seeds vs the oracle, 2,048 vs the reference
    wl = workloads.config4(count=1 << 16)
    idx = fm.build_index(wl.text, builder="gpu")
    ox = orc.OracleIndex(idx)
    seeds = workloads.unpack_patterns(wl.packed, 20)
    kl, _ = fm.exact_search_batch(idx, seeds)
    ours = _hits(idx, kl, 20, kl.shape[0])
    assert all(np.array_equal(a, b) for a, b in zip(ours, _oracle_hits(ox, kl, 20, kl.shape[0])))
    # the reference's set: config4(count=2048) (draws are per chunk of `count`, so a separate call)
    seeds = workloads.unpack_patterns(workloads.config4(count=1 << 11).packed, 20)
    kl, _ = fm.exact_search_batch(idx, seeds)
    for got, ref in zip(_per_pattern(*_hits(idx, kl, 20, kl.shape[0]), 2048), gold["config4_first2k_exact_hits"]):
        assert ref is None or [tuple(x) for x in ref] == got
    idx.release_device()
