"""Pin the CPU oracle (oracle/fm_oracle.c) against the reference's own outputs.

Fixtures in tests/golden were produced by running the reference package
itself (tests/golden/make_golden.py); known-answer values below are the
reference tests' own (cited).  The oracle reads indexes built by the native
builder, whose .fmi bytes are pinned to the reference in test_builder.py.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN, codes_to_str, small_text
from oracle import oracle as orc
from paper_1811_06127_b200 import build_index, workloads


@pytest.fixture(scope="module")
def acag():
    return orc.OracleIndex(build_index("ACAG"))


# tests/test_occ.py:14-20 (reference): occurrence table of "ACAG", rows 0..4
ACAG_OCC = [(0, 0, 1, 0), (0, 0, 1, 0), (0, 1, 1, 0), (1, 1, 1, 0), (2, 1, 1, 0)]


def test_oracle_acag_occ_table(acag):
    k = np.arange(5)
    out = orc.occ_pair_batch(acag, k, k)
    assert [tuple(r[4:]) for r in out] == ACAG_OCC
    # test_occ.py:86-99: occ_pair_all(2,4), (-1,4), ordering error
    out = orc.occ_pair_batch(acag, [2, -1], [4, 4])
    assert tuple(out[0]) == (0, 1, 1, 0, 2, 1, 1, 0)
    assert tuple(out[1]) == (0, 0, 0, 0, 2, 1, 1, 0)
    with pytest.raises(ValueError):
        orc.occ_pair_batch(acag, [3], [2])
    with pytest.raises(ValueError):
        orc.occ_pair_batch(acag, [0], [5])


def test_oracle_acag_search(acag):
    # test_search.py:48-53 (reference)
    kl = orc.exact_batch(acag, ["CA", "A", "ACAG", "T", "GG"])
    assert tuple(kl[0]) == (3, 3)
    assert tuple(kl[1]) == (1, 2)
    assert tuple(kl[2]) == (1, 1)
    assert kl[3, 0] > kl[3, 1] and kl[4, 0] > kl[4, 1]
    # test_search.py:104-107: inexact z=0 == exact; "T" has no match
    row, k, l, d, _ = orc.inexact_batch(acag, ["AG", "T"], 0)
    assert list(row) == [0, 1, 1] and (k[0], l[0], d[0]) == (2, 2, 0)
    # psi: test_search.py:200-208; locate: 236-240
    assert orc.psi(acag, 2) == (1, 3)
    assert orc.psi(acag, 1) is None
    assert list(orc.locate_batch(acag, np.arange(5))) == [4, 0, 2, 1, 3]


def test_oracle_small_cases(small_cases):
    for key, case in small_cases.items():
        n, seed = case["n"], case["seed"]
        idx = build_index(small_text(n, seed))
        ox = orc.OracleIndex(idx)
        occ = orc.occ_pair_batch(ox, case["occ_low"], case["occ_high"])
        assert np.array_equal(occ.astype(np.int64), np.array(case["occ"])), key
        kl = orc.exact_batch(ox, case["exact_patterns"])
        assert np.array_equal(kl, np.array(case["exact_kl"])), key
        for z in (0, 1, 2):
            sel = [i for i, zz in enumerate(case["inexact_z"]) if zz == z]
            if not sel:
                continue
            pats = [case["inexact_patterns"][i] for i in sel]
            row, k, l, d, _ = orc.inexact_batch(ox, pats, z)
            grow = case["inexact_row"]
            for j, i in enumerate(sel):
                a, b = grow[i], grow[i + 1]
                got = list(zip(k[row[j]:row[j + 1]], l[row[j]:row[j + 1]], d[row[j]:row[j + 1]]))
                want = list(zip(case["inexact_k"][a:b], case["inexact_l"][a:b], case["inexact_diffs"][a:b]))
                assert got == want, (key, pats[j], z)
        loc = orc.locate_batch(ox, np.arange(n + 1))
        assert list(loc) == case["locate"] == case["sa"], key
        for i in range(n + 1):
            p = orc.psi(ox, i)
            assert (list(p) if p else [-1, -1]) == case["psi"][i], (key, i)


def test_oracle_config0_full():
    meta = json.loads((GOLDEN / "config0_meta.json").read_text())
    wl = workloads.config0()
    import hashlib

    assert hashlib.sha256(wl.text.tobytes()).hexdigest() == meta["text_sha256"]
    assert hashlib.sha256(wl.patterns.tobytes()).hexdigest() == meta["patterns_sha256"]
    ox = orc.OracleIndex(build_index(wl.text))
    kl = orc.exact_batch(ox, wl.patterns)
    want = np.load(GOLDEN / "config0_exact.npz")["kl"].astype(np.int64)
    assert np.array_equal(kl, want)


def test_oracle_config1_head():
    path = GOLDEN / "config1_meta.json"
    if not path.exists():
        pytest.skip("config1 fixture not generated")
    wl = workloads.config1()
    ox = orc.OracleIndex(build_index(wl.text))
    head = np.load(GOLDEN / "config1_head.npz")["occ"]
    got = orc.occ_pair_batch(ox, wl.pairs[: head.shape[0], 0], wl.pairs[: head.shape[0], 1])
    assert np.array_equal(got, head)


@pytest.mark.slow
def test_oracle_config1_full_sha():
    import hashlib

    path = GOLDEN / "config1_meta.json"
    if not path.exists():
        pytest.skip("config1 fixture not generated")
    meta = json.loads(path.read_text())
    wl = workloads.config1()
    ox = orc.OracleIndex(build_index(wl.text))
    got = orc.occ_pair_batch(ox, wl.pairs[:, 0], wl.pairs[:, 1])
    assert hashlib.sha256(got.tobytes()).hexdigest() == meta["occ_sha256"]


def test_oracle_inexact_is_order_free_dedup(small_cases):
    """Results are unique by (k, l) and sorted by (k, l, diffs) (search.py:128-134, 153-159)."""
    idx = build_index(small_text(1000, 15))
    ox = orc.OracleIndex(idx)
    pats = [codes_to_str(small_text(8, s)) for s in range(40)]
    row, k, l, d, _ = orc.inexact_batch(ox, pats, 2)
    for j in range(len(pats)):
        kk, ll = k[row[j]:row[j + 1]], l[row[j]:row[j + 1]]
        keys = list(zip(kk, ll))
        assert keys == sorted(set(keys))


def test_oracle_config2_scale_golden():
    """Pins the oracle on the 64 Mbp config-2 genome: reference z = 1 result lists for the
    first 2000 seeds (tests/golden/make_golden.py scale, fmpm run on this text)."""
    cases = json.loads((GOLDEN / "scale_cases.json").read_text())["config2_first2k_z1"]
    wl = workloads.config2()
    ox = orc.OracleIndex(build_index(wl.text, builder="host"))
    row, k, l, d, _ = orc.inexact_batch(ox, wl.patterns[:2000], 1)
    for q, want in enumerate(cases):
        a, b = row[q], row[q + 1]
        assert list(zip(k[a:b].tolist(), l[a:b].tolist(), d[a:b].tolist())) == [tuple(x) for x in want], q
