"""The N-rank path on the GPU engine: two ranks (both on cuda:0, gloo
plumbing; no rank waits on another's kernels) each search their contiguous
shard, results are host-gathered (dist.gather_fixed / gather_csr) and must be
bit-identical to one rank searching everything; and `bench.py --gpus 2`
self-launches two ranks whose gathered digests agree."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, engine=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if engine:  # e.g. the flat z = 1 engine (the config-3 default at genome scale) forced on this small index
        os.environ["FMG_BIDIR_ENGINE"] = engine
    sys.path.insert(0, str(REPO))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1811_06127_b200 as fm
        from paper_1811_06127_b200 import workloads
        from paper_1811_06127_b200.dist import gather_csr, gather_fixed, shard_range

        wl = workloads.config2(n=6_000_000, n_reads=30_000)  # repeat genome, both strands, indels; bidirectional z = 1
        idx = fm.build_index(wl.text)
        pats = wl.patterns
        if engine == "flat":
            pats = np.ascontiguousarray(pats[:, :24])  # the flat engine takes patterns of at most 31 characters
        lo, hi = shard_range(pats.shape[0], rank, world)
        kl, _ = fm.exact_search_batch(idx, pats[lo:hi])
        ms = fm.inexact_search_batch(idx, pats[lo:hi], 1)
        pairs = workloads.occ_pairs(idx.n, 1 << 18, (11, 2))
        plo, phi = shard_range(pairs.shape[0], rank, world)
        occ = fm.occ_pair_batch(idx, pairs[plo:phi, 0], pairs[plo:phi, 1])
        all_kl = gather_fixed(kl, world)
        all_row, (all_k, all_l, all_d) = gather_csr(ms.offsets, [ms.k, ms.l, ms.diffs], world)
        all_occ = gather_fixed(occ, world)
        if rank == 0:
            fkl, _ = fm.exact_search_batch(idx, pats)
            fms = fm.inexact_search_batch(idx, pats, 1)
            focc = fm.occ_pair_batch(idx, pairs[:, 0], pairs[:, 1])
            ok = (np.array_equal(all_kl, fkl) and np.array_equal(all_row, fms.offsets)
                  and np.array_equal(all_k, fms.k) and np.array_equal(all_l, fms.l)
                  and np.array_equal(all_d, fms.diffs) and np.array_equal(all_occ, focc)
                  and all_row[-1] > 0)
            Path(out_dir, "ok").write_text("1" if ok else "0")
    finally:
        dist.destroy_process_group()


def test_two_engine_ranks_gather_equals_one_rank(gpu, tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").read_text() == "1"


def test_two_flat_engine_ranks_gather_equals_one_rank(gpu, tmp_path):
    """The same with the flat z = 1 engine (presence filter, chunk pipeline over the rank's own
    streams): each rank's engine caches and streams are its own, the gathered results one rank's."""
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), "flat"), nprocs=2, join=True)
    assert (tmp_path / "ok").read_text() == "1"


def test_bench_self_launches_two_ranks(gpu):
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--config", "config0",
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=str(REPO))
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["parity"]["ok"] is True and line["parity"]["ranks"] == 2
