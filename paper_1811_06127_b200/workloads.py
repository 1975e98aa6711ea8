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


def config4(count: int = 1 << 28, m: int = 20, n: int = 1_000_000_000) -> Workload:
    """High-batch exact seeds: 1 Gbp i.i.d. (seed 5); 80% exact substrings, 20% random."""
    text = iid_text(n, 5)
    q = _rng(5, 1)
    exact = q.random(count) < 0.8
    pats = q.integers(0, 4, size=(count, m), dtype=np.uint8)
    ne = int(exact.sum())
    offs = q.integers(0, n - m + 1, size=ne)
    pats[exact] = substrings(text, offs, m)
    return Workload("config4", text, patterns=pats, meta={"m": m})


CONFIGS = {"config0": config0, "config1": config1, "config1h": config1h, "config2": config2,
           "config4": config4}
