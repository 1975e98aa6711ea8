"""CLI on the GPU: byte-identical TSV / stderr to the reference CLI (tests/golden/cli)."""

import subprocess
import sys

import pytest

from conftest import GOLDEN, REPO
from paper_1811_06127_b200.cli import EXIT_OK, main

pytestmark = pytest.mark.gpu
CLI = GOLDEN / "cli"


@pytest.fixture(scope="module")
def fmi(tmp_path_factory, gpu):
    out = tmp_path_factory.mktemp("cli") / "ref.fmi"
    assert main(["index", str(CLI / "ref.fa"), "-o", str(out)]) == EXIT_OK
    return out


@pytest.mark.parametrize("name,extra", [("match_z0", ["-z", "0"]), ("match_z1", ["-z", "1"]),
                                        ("match_z2", ["-z", "2"]), ("match_max2", ["-z", "1", "--max-hits", "2"])])
def test_match_byte_identical(fmi, capsys, name, extra):
    assert main(["match", str(fmi), "-f", str(CLI / "patterns.txt"), *extra]) == EXIT_OK
    cap = capsys.readouterr()
    assert cap.out == (CLI / f"{name}.out").read_text()
    assert cap.err == (CLI / f"{name}.err").read_text()


def test_bench_checksum_matches_reference(fmi, capsys):
    assert main(["bench", str(fmi), "--iters", "30", "--seed", "3"]) == EXIT_OK
    cap = capsys.readouterr()
    lines = [ln.split("\t") for ln in cap.out.strip().splitlines()]
    ref = (CLI / "bench.out").read_text().strip().split("\t")
    # one line per concrete kernel (the reference's default list), all on the GPU
    assert [ln[0] for ln in lines] == ["scalar", "bytelut", "nibble", "simd"]
    assert all(ln[5] == ref[5] for ln in lines)
    assert "answer checksums agree" in cap.err


def test_reference_cli_examples(tmp_path, capsys):
    # reference tests/test_cli.py:17-29, 83-94, 135-144
    fa = tmp_path / "acag.fa"
    fa.write_text(">r1\nACAG\n")
    fmi = tmp_path / "acag.fmi"
    assert main(["index", str(fa), "-o", str(fmi)]) == EXIT_OK
    capsys.readouterr()
    assert main(["match", str(fmi), "-p", "CA", "-z", "0"]) == EXIT_OK
    assert capsys.readouterr().out == "0\tr1\t1\t0\n"
    assert main(["match", str(fmi), "-p", "AT", "-z", "1"]) == EXIT_OK
    assert capsys.readouterr().out == "0\tr1\t0\t1\n0\tr1\t2\t1\n"
    assert main(["match", str(fmi), "-p", "ANA"]) == EXIT_OK
    cap = capsys.readouterr()
    assert cap.out == "" and "non-ACGT" in cap.err
    two = tmp_path / "two.fa"
    two.write_text(">r1\nAAACCC\n>r2\nGGGTTT\n")
    fmi2 = tmp_path / "two.fmi"
    assert main(["index", str(two), "-o", str(fmi2)]) == EXIT_OK
    capsys.readouterr()
    assert main(["match", str(fmi2), "-p", "GGG"]) == EXIT_OK
    assert capsys.readouterr().out == "0\tr2\t0\t0\n"
    assert main(["match", str(fmi2), "-p", "CCGG"]) == EXIT_OK
    assert capsys.readouterr().out == ""
    proc = subprocess.run([sys.executable, "-m", "paper_1811_06127_b200", "match", str(fmi), "-p", "CA"],
                          capture_output=True, text=True, cwd=str(REPO))
    assert proc.returncode == EXIT_OK and proc.stdout == "0\tr1\t1\t0\n"
