"""Deterministic synthetic workloads for BASELINE.json configs 0-4.

No public dataset is used: every text and query set is drawn from numpy's
PCG64 with a fixed seed and a fixed draw order, so the GPU path, the CPU
oracle and the reference all consume identical bytes.  Ambiguities in the
config text are resolved as documented in DESIGN.md §6.

Streams: the text of config `i` uses PCG64(seed); its queries use
PCG64([seed, 1]); auxiliary draws use PCG64([seed, 2]) and up.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GC_41 = np.array([0.295, 0.205, 0.205, 0.295])  # A, C, G, T at 41% GC


def _rng(*seed) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(list(seed) if len(seed) > 1 else seed[0]))


@dataclass
class Workload:
    name: str
    text: np.ndarray                       # uint8 codes in [0, 4)
    patterns: np.ndarray | None = None     # (N, m) uint8 codes, fixed length
    packed: np.ndarray | None = None       # (N,) uint64 2-bit packed patterns (m <= 32)
    pairs: np.ndarray | None = None        # (N, 2) int64 (low, high) = (k-1, l)
    max_diff: int = 0
    meta: dict = field(default_factory=dict)


def iid_text(n: int, seed: int, probs=None) -> np.ndarray:
    rng = _rng(seed)
    if probs is None:
        return rng.integers(0, 4, size=n, dtype=np.uint8)
    return rng.choice(4, size=n, p=probs).astype(np.uint8)


def substrings(text: np.ndarray, offsets: np.ndarray, m: int) -> np.ndarray:
    return text[offsets[:, None] + np.arange(m)[None, :]]


def config0(n_patterns: int = 10_000, m: int = 32) -> Workload:
    """Exact search: 1 Mbp i.i.d. (seed 42); even ids exact substrings, odd ids random."""
    text = iid_text(1_000_000, 42)
    q = _rng(42, 1)
    half = n_patterns // 2
    offs = q.integers(0, text.size - m + 1, size=n_patterns - half)
    pats = np.empty((n_patterns, m), dtype=np.uint8)
    pats[0::2] = substrings(text, offs, m)
    pats[1::2] = q.integers(0, 4, size=(half, m), dtype=np.uint8)
    return Workload("config0", text, patterns=pats, meta={"m": m})


def occ_pairs(n: int, count: int, seed) -> np.ndarray:
    """(low, high) = (k-1, l): k ~ U{0..n}, l = min(n, k + Geometric(0.01))."""
    q = _rng(*seed) if isinstance(seed, tuple) else _rng(seed)
    k = q.integers(0, n + 1, size=count, dtype=np.int64)
    g = q.geometric(0.01, size=count).astype(np.int64)
    l = np.minimum(n, k + g)
    return np.stack([k - 1, l], axis=1)


def config1(count: int = 1 << 24, shard: int = 0) -> Workload:
    """Occ microbenchmark: 2^24-base i.i.d. text (seed 7), 2^24 (k-1, l) pairs.

    `shard` > 0 draws an independent pair set of the same distribution (used
    for weak scaling: rank r processes shard r).
    """
    text = iid_text(1 << 24, 7)
    seed = (7, 1) if shard == 0 else (7, 1, shard)
    return Workload("config1", text, pairs=occ_pairs(text.size, count, seed))


def config1h(count: int = 1 << 24, n: int = 1_000_000_000) -> Workload:
    """Config 1's pair distribution over config 4's 1 Gbp text (HBM-resident index)."""
    text = iid_text(n, 5)
    return Workload("config1h", text, pairs=occ_pairs(n, count, (5, 3)))


def mutate(seq: np.ndarray, rate: float, rng: np.random.Generator) -> np.ndarray:
    """Independent substitutions: each base replaced by a different base with prob `rate`."""
    out = seq.copy()
    hit = rng.random(seq.size) < rate
    shift = rng.integers(1, 4, size=int(hit.sum()), dtype=np.uint8)
    out[hit] = (out[hit] + shift) % 4
    return out


def revcomp(codes: np.ndarray) -> np.ndarray:
    return (3 - codes[..., ::-1]).astype(np.uint8)


def repeat_genome(n: int, seed: int, n_elements: int, element_len: int, fraction: float,
                  divergence: float) -> np.ndarray:
    """GC-41% background with `fraction` of bases covered by diverged element copies.

    Copies are forward-strand, one per equal slot of n / n_copies bases at a
    uniform offset inside the slot, elements assigned round-robin.
    """
    text = iid_text(n, seed, GC_41)
    aux = _rng(seed, 2)
    elements = aux.choice(4, size=(n_elements, element_len), p=GC_41).astype(np.uint8)
    n_copies = int(round(fraction * n / element_len))
    slot = n // n_copies
    starts = np.arange(n_copies, dtype=np.int64) * slot + aux.integers(0, slot - element_len + 1, size=n_copies)
    for e in range(n_elements):
        idx = np.arange(e, n_copies, n_elements)
        copies = np.broadcast_to(elements[e], (idx.size, element_len)).reshape(-1)
        copies = mutate(copies, divergence, aux).reshape(idx.size, element_len)
        pos = starts[idx][:, None] + np.arange(element_len)[None, :]
        text[pos] = copies
    return text


def sample_reads(text: np.ndarray, count: int, length: int, sub_rate: float, indel_rate: float,
                 rng: np.random.Generator) -> np.ndarray:
    """Reads from uniform positions and strands with substitution/indel errors.

    A window of length + 8 is drawn, substitutions applied per base, then each
    base independently suffers an indel with prob `indel_rate` (insertion of a
    random base or deletion, equally likely); the read is cut to `length`.
    """
    win = length + 8
    pos = rng.integers(0, text.size - win + 1, size=count, dtype=np.int64)
    strand = rng.integers(0, 2, size=count).astype(bool)
    reads = substrings(text, pos, win)
    reads[strand] = revcomp(reads[strand])
    reads = mutate(reads.reshape(-1), sub_rate, rng).reshape(count, win)
    has_indel = rng.random((count, win)) < indel_rate
    out = np.empty((count, length), dtype=np.uint8)
    plain = ~has_indel.any(axis=1)
    out[plain] = reads[plain, :length]
    for r in np.flatnonzero(~plain):
        seq = []
        for j in range(win):
            if has_indel[r, j]:
                if rng.random() < 0.5:
                    seq.append(int(rng.integers(0, 4)))
                    seq.append(int(reads[r, j]))
                # deletion: drop the base
            else:
                seq.append(int(reads[r, j]))
        seq = (seq + [0] * length)[:length]
        out[r] = seq
    return out


def config2(n_reads: int = 1_000_000, n: int = 64_000_000) -> Workload:
    """Inexact z=1: 64 Mbp repeat genome (seed 3), 32-bp seed prefixes of 100-bp reads."""
    text = repeat_genome(n, 3, n_elements=20, element_len=300, fraction=0.30, divergence=0.10)
    reads = sample_reads(text, n_reads, 100, 0.01, 0.0005, _rng(3, 1))
    return Workload("config2", text, patterns=np.ascontiguousarray(reads[:, :32]), max_diff=1,
                    meta={"read_len": 100, "seed_len": 32})


def pack_substrings(text, offsets: np.ndarray, m: int) -> np.ndarray:
    """2-bit packed text[o : o+m] for each offset (char j in bits 2j..2j+1).

    `text` may be a CUDA tensor copy of the text (same result, faster gathers).
    """
    if hasattr(text, "is_cuda"):
        import torch

        o = torch.from_numpy(offsets.astype(np.int64)).to(text.device)
        acc = torch.zeros(offsets.size, dtype=torch.int64, device=text.device)
        for j in range(m):
            acc |= text[o + j].to(torch.int64) << (2 * j)
        return acc.cpu().numpy().view(np.uint64)
    out = np.zeros(offsets.size, dtype=np.uint64)
    for j in range(m):
        out |= text[offsets + j].astype(np.uint64) << np.uint64(2 * j)
    return out


def unpack_patterns(packed: np.ndarray, m: int) -> np.ndarray:
    """(N,) packed uint64 -> (N, m) uint8 codes."""
    shifts = (2 * np.arange(m, dtype=np.uint64))[None, :]
    return ((packed[:, None] >> shifts) & np.uint64(3)).astype(np.uint8)


def config4(count: int = 1 << 28, m: int = 20, n: int = 1_000_000_000, chunk: int = 1 << 22) -> Workload:
    """High-batch exact seeds: 1 Gbp i.i.d. (seed 5); 80% exact substrings, 20% random.

    Generated in chunks of `chunk` seeds directly as 2-bit packed words: per
    chunk, a Bernoulli(0.8) exact flag, a uniform random packed m-mer and a
    uniform text offset are drawn (in that order); exact seeds take the text.
    """
    text = iid_text(n, 5)
    src = text
    try:  # gathers on the GPU when there is one (identical bytes)
        import torch

        if torch.cuda.is_available():
            src = torch.from_numpy(text).cuda()
    except ImportError:  # pragma: no cover
        pass
    q = _rng(5, 1)
    packed = np.empty(count, dtype=np.uint64)
    for c0 in range(0, count, chunk):
        c = min(chunk, count - c0)
        exact = q.random(c) < 0.8
        rand = q.integers(0, 4 ** m, size=c, dtype=np.uint64)
        offs = q.integers(0, n - m + 1, size=c)
        rand[exact] = pack_substrings(src, offs[exact], m)
        packed[c0:c0 + c] = rand
    del src
    return Workload("config4", text, packed=packed, meta={"m": m})


# Markov-1 background of config 3: rows = previous base, columns = next base,
# CpG-depleted; stationary distribution ~(0.296, 0.207, 0.208, 0.289) = 41.5% GC.
MARKOV1 = np.array([[0.33, 0.17, 0.24, 0.26],
                    [0.36, 0.27, 0.05, 0.32],
                    [0.29, 0.22, 0.26, 0.23],
                    [0.22, 0.19, 0.25, 0.34]])


MARKOV_CHUNK = 1 << 26  # bases per independently seeded chunk (fixed: output does not depend on workers)


def _markov_chunk(args) -> np.ndarray:
    seed, c, size, segment = args
    rng = _rng(seed, 10, c)
    # transition table over (previous base, u8): P quantised to 1/256
    cum = np.cumsum(MARKOV1 / MARKOV1.sum(1, keepdims=True), axis=1)
    u = (np.arange(256) + 0.5) / 256.0
    table = np.array([[int((uu > cum[prev, :3]).sum()) for uu in u] for prev in range(4)],
                     dtype=np.uint8).reshape(-1)
    n_seg = (size + segment - 1) // segment
    out = np.empty((segment, n_seg), dtype=np.uint8)
    state = rng.choice(4, size=n_seg, p=GC_41).astype(np.uint16)
    out[0] = state
    for j in range(1, segment):
        state = table[(state << 8) | rng.integers(0, 256, size=n_seg, dtype=np.uint16)].astype(np.uint16)
        out[j] = state
    return np.ascontiguousarray(out.T).reshape(-1)[:size]


def markov1_text(n: int, seed: int, segment: int = 4096, workers: int | None = None) -> np.ndarray:
    """Markov-1 text (matrix MARKOV1, transitions quantised to 1/256) generated as
    independent `segment`-base chains, each starting from the GC-41%
    distribution; chunks of MARKOV_CHUNK bases use their own PCG64 streams and
    run in parallel processes."""
    import multiprocessing as mp
    import os

    jobs = [(seed, c, min(MARKOV_CHUNK, n - c * MARKOV_CHUNK), segment)
            for c in range((n + MARKOV_CHUNK - 1) // MARKOV_CHUNK)]
    workers = workers or min(len(jobs), len(os.sched_getaffinity(0)))
    if workers <= 1 or len(jobs) == 1:
        parts = [_markov_chunk(j) for j in jobs]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            parts = pool.map(_markov_chunk, jobs)
    return np.concatenate(parts)


def family_genome(n: int, seed: int, n_families: int = 500, len_range=(100, 6000), fraction: float = 0.45,
                  div_range=(0.05, 0.20)) -> np.ndarray:
    """Config 3 genome: Markov-1 background with `fraction` of it overwritten by
    interspersed copies of `n_families` random elements (lengths uniform in
    len_range, per-copy substitution divergence uniform in div_range).  Copies
    are forward-strand, one per equal slot at a uniform offset inside the slot;
    families are drawn uniformly per copy."""
    text = markov1_text(n, seed)
    aux = _rng(seed, 2)
    lens = aux.integers(len_range[0], len_range[1] + 1, size=n_families)
    fams = [aux.choice(4, size=int(L), p=GC_41).astype(np.uint8) for L in lens]
    n_copies = int(round(fraction * n / lens.mean()))
    slot = n // n_copies
    fam_of = aux.integers(0, n_families, size=n_copies)
    fam_of = np.where(lens[fam_of] <= slot, fam_of, int(np.argmin(lens)))
    div = aux.uniform(div_range[0], div_range[1], size=n_copies)
    off = (aux.random(n_copies) * (slot - lens[fam_of] + 1)).astype(np.int64)
    starts = np.arange(n_copies, dtype=np.int64) * slot + off
    for f in range(n_families):
        idx = np.flatnonzero(fam_of == f)
        if idx.size == 0:
            continue
        L = int(lens[f])
        copies = np.broadcast_to(fams[f], (idx.size, L)).copy()
        hit = aux.random((idx.size, L)) < div[idx][:, None]
        shift = aux.integers(1, 4, size=int(hit.sum()), dtype=np.uint8)
        copies[hit] = (copies[hit] + shift) % 4
        pos = starts[idx][:, None] + np.arange(L)[None, :]
        text[pos] = copies
    return text


_C3_TEXT = None  # shared with forked workers (copy-on-write)


def _config3_chunk(args) -> np.ndarray:
    c, count, read_len, seed_len, stride = args
    rng = _rng(11, 1, c)
    offs = np.arange(0, read_len - seed_len + 1, stride)
    reads = sample_reads(_C3_TEXT, count, read_len, 0.005, 0.0, rng)
    out = np.zeros(count * offs.size, dtype=np.uint64).reshape(count, offs.size)
    for j in range(seed_len):
        out |= reads[:, offs + j].astype(np.uint64) << np.uint64(2 * j)
    return out.reshape(-1)


def config3(n_reads: int = 10_000_000, n: int = 3_100_000_000, read_len: int = 150, seed_len: int = 19,
            stride: int = 10, workers: int | None = None) -> Workload:
    """Genome-scale seeds: 3.1 Gbp family genome (seed 11); 10M x 150-bp reads with
    0.5% substitutions from both strands; 19-bp seeds at offsets 0, 10, ..., 130
    (14 per read), 2-bit packed, read-major.  Reads are drawn in chunks of 2^20
    with streams PCG64([11, 1, chunk]) in parallel processes."""
    import multiprocessing as mp
    import os

    global _C3_TEXT
    text = family_genome(n, 11)
    chunk = 1 << 20
    jobs = [(c, min(chunk, n_reads - c * chunk), read_len, seed_len, stride)
            for c in range((n_reads + chunk - 1) // chunk)]
    _C3_TEXT = text
    try:
        workers = workers or min(len(jobs), len(os.sched_getaffinity(0)))
        if workers <= 1 or len(jobs) == 1:
            parts = [_config3_chunk(j) for j in jobs]
        else:
            with mp.get_context("fork").Pool(workers) as pool:
                parts = pool.map(_config3_chunk, jobs)
    finally:
        _C3_TEXT = None
    packed = np.concatenate(parts)
    n_seeds = (read_len - seed_len) // stride + 1
    return Workload("config3", text, packed=packed, max_diff=1,
                    meta={"m": seed_len, "reads": n_reads, "seeds_per_read": n_seeds})


CONFIGS = {"config0": config0, "config1": config1, "config1h": config1h, "config2": config2,
           "config3": config3, "config4": config4}
