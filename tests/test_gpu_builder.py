"""GPU index builder (fmb_build_gpu) vs the host SA-IS builder and the reference's .fmi bytes."""

import hashlib
import io
import json

import numpy as np
import pytest

import paper_1811_06127_b200 as fm
from conftest import GOLDEN, small_text
from paper_1811_06127_b200 import workloads

pytestmark = pytest.mark.gpu


def fmi(index) -> bytes:
    buf = io.BytesIO()
    fm.serialize_index(index, buf)
    return buf.getvalue()


def test_gpu_builder_small_cases(small_cases, gpu):
    for key, case in small_cases.items():
        idx = fm.build_index(small_text(case["n"], case["seed"]), builder="gpu")
        assert hashlib.sha256(fmi(idx)).hexdigest() == case["fmi_sha256"], key


def test_gpu_builder_repetitive_texts(gpu):
    rng = np.random.Generator(np.random.PCG64(31))
    texts = [np.zeros(5000, np.uint8), np.tile(np.array([0, 1], np.uint8), 3000),
             np.tile(rng.integers(0, 4, 37, dtype=np.uint8), 400), rng.integers(0, 4, 100_000, dtype=np.uint8),
             np.concatenate([np.tile(rng.integers(0, 4, 300, dtype=np.uint8), 50),
                             rng.integers(0, 4, 7000, dtype=np.uint8)])]
    for t in texts:
        assert fm.build_index(t, builder="gpu") == fm.build_index(t, builder="host")


def test_gpu_builder_config_fmi():
    for name, meta in (("config0", "config0_meta.json"), ("config1", "config1_meta.json")):
        wl = getattr(workloads, name)()
        want = json.loads((GOLDEN / meta).read_text())["fmi_sha256"]
        assert hashlib.sha256(fmi(fm.build_index(wl.text, builder="gpu"))).hexdigest() == want, name


def test_gpu_builder_repeat_genome_matches_host():
    text = workloads.repeat_genome(4_000_000, 3, n_elements=20, element_len=300, fraction=0.3, divergence=0.1)
    assert fm.build_index(text, builder="gpu") == fm.build_index(text, builder="host")
