"""Native index builder and .fmi I/O vs the reference (host only, no GPU).

The .fmi written from the native SA-IS build must be byte-identical to the
reference's serialize_index(build_index(text)) (fixtures: SHA-256 of the
reference's bytes), which pins the BWT, sentinel row, C table, bucket bases,
padding and suffix-array samples at once.
"""

import hashlib
import io
import json

import numpy as np
import pytest

from conftest import GOLDEN, small_text
from paper_1811_06127_b200 import (
    BadMagicError,
    ChecksumError,
    FmIndex,
    IndexFormatError,
    RecordSpan,
    TruncatedStreamError,
    VersionMismatchError,
    build_c_table,
    build_index,
    check_index,
    deserialize_index,
    serialize_index,
    suffix_array,
    workloads,
)


def fmi(index) -> bytes:
    buf = io.BytesIO()
    n = serialize_index(index, buf)
    assert n == len(buf.getvalue())
    return buf.getvalue()


def test_small_fmi_byte_identical(small_cases):
    for key, case in small_cases.items():
        idx = build_index(small_text(case["n"], case["seed"]))
        assert hashlib.sha256(fmi(idx)).hexdigest() == case["fmi_sha256"], key
        assert list(suffix_array(small_text(case["n"], case["seed"]))) == case["sa"], key
        check_index(idx)


def test_config0_fmi_byte_identical():
    meta = json.loads((GOLDEN / "config0_meta.json").read_text())
    idx = build_index(workloads.config0().text)
    assert hashlib.sha256(fmi(idx)).hexdigest() == meta["fmi_sha256"]


def test_config1_fmi_byte_identical():
    path = GOLDEN / "config1_meta.json"
    if not path.exists():
        pytest.skip("config1 fixture not generated")
    meta = json.loads(path.read_text())
    idx = build_index(workloads.config1().text)
    assert hashlib.sha256(fmi(idx)).hexdigest() == meta["fmi_sha256"]


def test_acag_worked_example():
    # reference test_acceptance.py:95-110 / test_index.py:33-41
    assert list(suffix_array("ACAG")) == [4, 0, 2, 1, 3]
    idx = build_index("ACAG")
    assert idx.n == 4 and idx.c == (0, 2, 3, 4, 4) and idx.sentinel_row == 1
    assert len(idx.buckets) == 1 and tuple(idx.sa_samples) == (4,)
    assert idx.records == (RecordSpan(name="ref", start=0, length=4),)
    check_index(idx)


def test_single_character_and_lowercase():
    idx = build_index("A")
    assert idx.n == 1 and idx.c == (0, 1, 1, 1, 1) and tuple(idx.sa_samples) == (1,)
    assert fmi(build_index("acgtAC")) == fmi(build_index("ACGTAC"))


def test_build_rejects_bad_input():
    with pytest.raises(ValueError):
        build_index("")
    with pytest.raises(ValueError):
        build_index("ACGN")
    with pytest.raises(ValueError):
        build_index("ACGT", [("r1", 0, 3)])
    with pytest.raises(ValueError):
        build_index("ACGT", [("", 0, 4)])


def test_c_table_examples():
    assert build_c_table([2, 1, 1, 0]) == (0, 2, 3, 4, 4)
    with pytest.raises(ValueError):
        build_c_table([1, 2, 3])


def test_round_trip_and_records():
    idx = build_index("ACGTACGT", [("r1", 0, 3), ("r2", 3, 5)])
    back = deserialize_index(io.BytesIO(fmi(idx)))
    assert back == idx and [r.name for r in back.records] == ["r1", "r2"]
    check_index(back)


def test_final_bucket_padding_zero():
    idx = build_index(small_text(128, 10))
    assert len(idx.buckets) == 2 and set(idx.buckets[1].chars[1:]) == {0}


def test_check_index_catches_tampering():
    idx = build_index(small_text(150, 3))
    rec = idx.bucket_records.copy()
    rec[1, :32] = 0
    broken = FmIndex(idx.n, idx.c, rec, idx.sentinel_row, idx.sa_samples, idx.records)
    with pytest.raises(ValueError, match="telescoping"):
        check_index(broken)
    broken = FmIndex(idx.n, (0, 1, 2, 3, 5), idx.bucket_records, idx.sentinel_row, idx.sa_samples,
                     idx.records)
    with pytest.raises(ValueError):
        check_index(broken)


def test_format_errors():
    data = fmi(build_index(small_text(300, 14)))
    with pytest.raises(BadMagicError):
        deserialize_index(io.BytesIO(b"XXXX" + data[4:]))
    with pytest.raises(VersionMismatchError):
        deserialize_index(io.BytesIO(data[:4] + b"\x02\x00" + data[6:]))
    with pytest.raises(TruncatedStreamError):
        deserialize_index(io.BytesIO(data[:200]))
    with pytest.raises(TruncatedStreamError):
        deserialize_index(io.BytesIO(data[:-2]))
    flipped = bytearray(data)
    flipped[100] ^= 0xFF
    with pytest.raises(ChecksumError):
        deserialize_index(io.BytesIO(bytes(flipped)))
    bad = bytearray(data)
    bad[16] = 64  # bucket size witness
    with pytest.raises(IndexFormatError):
        deserialize_index(io.BytesIO(bytes(bad)))


def test_suffix_array_properties_random():
    rng = np.random.Generator(np.random.PCG64(77))
    for n in (2, 17, 200, 5000):
        for kind in range(3):
            if kind == 0:
                codes = rng.integers(0, 4, n, dtype=np.uint8)
            elif kind == 1:
                codes = np.zeros(n, dtype=np.uint8)
            else:
                codes = np.tile(rng.integers(0, 4, 7, dtype=np.uint8), n // 7 + 1)[:n]
            sa = suffix_array(codes)
            text = bytes(codes + 1) + b"\x00"
            keys = [text[i:] for i in sa]
            assert keys == sorted(keys)
            assert sorted(sa.tolist()) == list(range(n + 1))
