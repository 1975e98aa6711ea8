"""FASTA ingestion and the CLI front-end on the host (no GPU needed).

Cases follow the reference's tests/test_fasta.py and tests/test_cli.py; the
`index` command must write the reference's exact .fmi bytes.
"""

import hashlib
import io

import pytest

from conftest import GOLDEN
from paper_1811_06127_b200.cli import EXIT_CORRUPT, EXIT_IO, EXIT_OK, EXIT_USAGE, main
from paper_1811_06127_b200.fasta import FastaError, FastaRecord, read_fasta

CLI = GOLDEN / "cli"


def test_fasta_records_and_folding():
    assert read_fasta(io.StringIO(">r1\nACAG\n")) == [FastaRecord("r1", "ACAG", 0)]
    recs = read_fasta(io.StringIO(">r1 description here\nacg\nT\n\nACGT\n"))
    assert recs[0].name == "r1" and recs[0].sequence == "ACGTACGT"
    recs = read_fasta(io.StringIO(">a\nAC\n>b\nGT\n"))
    assert [r.sequence for r in recs] == ["AC", "GT"]


def test_fasta_errors():
    with pytest.raises(FastaError, match=r"'r1'.*'N' at offset 2"):
        read_fasta(io.StringIO(">r1\nACNG\n"))
    with pytest.raises(FastaError, match="offset 5"):
        read_fasta(io.StringIO(">r1\nACGT\nAN\n"))
    for bad in ("", "\n\n", "ACGT\n", ">\nACGT\n"):
        with pytest.raises(FastaError):
            read_fasta(io.StringIO(bad))
    with pytest.raises(FastaError, match="empty sequence"):
        read_fasta(io.StringIO(">r1\n>r2\nAC\n"))


def test_fasta_sanitize():
    recs = read_fasta(io.StringIO(">r1\nACNGN\n>r2\nGGT\n"), sanitize=True)
    assert recs[0].sequence == "ACAGA" and recs[0].substituted == 2 and recs[1].substituted == 0


def test_index_command_writes_reference_bytes(tmp_path, capsys):
    out = tmp_path / "ref.fmi"
    assert main(["index", str(CLI / "ref.fa"), "-o", str(out)]) == EXIT_OK
    assert hashlib.sha256(out.read_bytes()).hexdigest() == (CLI / "ref.fmi.sha256").read_text()
    assert capsys.readouterr().err == (CLI / "index.err").read_text()


def test_usage_io_and_corrupt_errors(tmp_path, capsys):
    fa = tmp_path / "ref.fa"
    fa.write_text(">r1\nACAG\n")
    fmi = tmp_path / "ref.fmi"
    assert main(["index", str(fa), "-o", str(fmi)]) == EXIT_OK
    assert main(["match", str(fmi)]) == EXIT_USAGE
    assert main(["match", str(fmi), "-p", "CA", "-z", "-1"]) == EXIT_USAGE
    assert main(["match", str(fmi), "-p", ""]) == EXIT_USAGE
    assert main(["nonsense"]) == EXIT_USAGE
    assert main(["match", str(fmi), "-p", "CA", "--kernel", "bogus"]) == EXIT_USAGE
    assert main(["index", str(tmp_path / "missing.fa"), "-o", str(tmp_path / "x.fmi")]) == EXIT_IO
    assert main(["match", str(tmp_path / "missing.fmi"), "-p", "CA"]) == EXIT_IO
    blob = bytearray(fmi.read_bytes())
    blob[-2] ^= 0xFF
    (tmp_path / "bad.fmi").write_bytes(bytes(blob))
    assert main(["match", str(tmp_path / "bad.fmi"), "-p", "CA"]) == EXIT_CORRUPT
    (tmp_path / "bogus.fmi").write_bytes(b"this is not an index file at all")
    assert main(["match", str(tmp_path / "bogus.fmi"), "-p", "CA"]) == EXIT_CORRUPT
    bad = tmp_path / "bad.fa"
    bad.write_text(">r1\nACNG\n")
    capsys.readouterr()
    assert main(["index", str(bad), "-o", str(tmp_path / "y.fmi")]) == EXIT_USAGE
    assert "offset 2" in capsys.readouterr().err


def test_match_without_gpu_fails_loudly(tmp_path, capsys):
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    fa = tmp_path / "ref.fa"
    fa.write_text(">r1\nACAG\n")
    fmi = tmp_path / "ref.fmi"
    assert main(["index", str(fa), "-o", str(fmi)]) == EXIT_OK
    capsys.readouterr()
    assert main(["match", str(fmi), "-p", "CA"]) == EXIT_IO
    assert "no CUDA device" in capsys.readouterr().err
