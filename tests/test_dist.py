"""Multi-rank plumbing on CPU (gloo, world size 2): query sharding and the host gather.

The per-rank engine here is the CPU oracle (test infrastructure), standing in
for the GPU kernels, which the GPU tests cover; what is tested is that the
shards tile the query set and the gathered results equal the single-rank run.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_06127_b200.dist import gather_csr, gather_fixed, max_over_ranks, shard_range


def test_shard_range_tiles():
    for count in (0, 1, 7, 1000, 12345):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as orc
        from paper_1811_06127_b200 import build_index

        rng = np.random.Generator(np.random.PCG64(5))
        text = rng.integers(0, 4, 20_000, dtype=np.uint8)
        idx = build_index(text, builder="host")
        ox = orc.OracleIndex(idx)
        pats = rng.integers(0, 4, (301, 12), dtype=np.uint8)
        lo, hi = shard_range(pats.shape[0], rank, world)
        kl = orc.exact_batch(ox, pats[lo:hi], threads=1)
        all_kl = gather_fixed(kl, world)
        u32 = gather_fixed(kl.astype(np.uint32), world)  # gloo has no uint32: shipped as int32 bytes
        assert u32.dtype == np.uint32 and np.array_equal(u32, all_kl.astype(np.uint32))
        row, k, l, d, _ = orc.inexact_batch(ox, pats[lo:hi], 1, threads=1)
        all_row, (all_k, all_l, all_d) = gather_csr(row, [k, l, d], world)
        t = max_over_ranks(float(rank + 1), world)
        if rank == 0:
            full_kl = orc.exact_batch(ox, pats, threads=1)
            frow, fk, fl, fd, _ = orc.inexact_batch(ox, pats, 1, threads=1)
            ok = (np.array_equal(all_kl, full_kl) and np.array_equal(all_row, frow)
                  and np.array_equal(all_k, fk) and np.array_equal(all_l, fl) and np.array_equal(all_d, fd)
                  and t == float(world))
            with open(os.path.join(out_dir, "ok"), "w") as f:
                f.write("1" if ok else "0")
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert (tmp_path / "ok").read_text() == "1"
