"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container, where the reference is mounted read-only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py small config0 config1

Every fixture records the reference's own outputs (fmpm from
/root/reference/pkg/src) on seeded inputs that the tests regenerate
bit-identically (numpy PCG64 / workloads.py).  Large outputs are pinned by
SHA-256; small ones are stored in full.  Nothing here runs on the GPU box:
/root/reference does not exist there, only these committed fixtures travel.
"""

from __future__ import annotations

import hashlib
import io
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import fmpm  # noqa: E402  (the reference)

from paper_1811_06127_b200 import workloads  # noqa: E402

SYM = np.array(list("ACGT"))


def text_of(codes: np.ndarray) -> str:
    return "".join(SYM[codes].tolist())


def sha(a) -> str:
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a).tobytes()
    return hashlib.sha256(a).hexdigest()


def fmi_bytes(index) -> bytes:
    buf = io.BytesIO()
    fmpm.serialize_index(index, buf)
    return buf.getvalue()


# (n, seed) of the small random texts; sizes straddle bucket (128), line (64)
# and sample (32) boundaries
SMALL = [(1, 1), (4, 2), (31, 3), (32, 4), (33, 5), (63, 6), (64, 7), (65, 8), (127, 9), (128, 10),
         (129, 11), (255, 12), (256, 13), (300, 14), (1000, 15), (2500, 16)]


def small_text(n: int, seed: int) -> np.ndarray:
    return np.random.Generator(np.random.PCG64([900, seed])).integers(0, 4, n, dtype=np.uint8)


def gen_small():
    out = {}
    for n, seed in SMALL:
        codes = small_text(n, seed)
        text = text_of(codes)
        idx = fmpm.build_index(text)
        rng = np.random.Generator(np.random.PCG64([901, seed]))
        # Occ pairs: random plus every edge case of occ.py:59-96
        low = rng.integers(-1, n + 1, 300)
        high = np.minimum(n, low + rng.geometric(0.05, 300))
        extra = [(-1, -1), (-1, 0), (-1, n), (0, 0), (n, n), (0, n), (n - 1 if n else 0, n)]
        low = np.concatenate([low, [a for a, _ in extra]])
        high = np.concatenate([high, [b for _, b in extra]])
        occ = np.array([tuple(p.at_low) + tuple(p.at_high)
                        for p in (fmpm.occ_pair_all(idx, int(a), int(b)) for a, b in zip(low, high))],
                       dtype=np.int64)
        # exact patterns: present substrings and random, lengths 1..40
        pats = []
        for _ in range(200):
            m = int(rng.integers(1, 41))
            if rng.random() < 0.6 and m <= n:
                s = int(rng.integers(0, n - m + 1))
                pats.append(text[s:s + m])
            else:
                pats.append(text_of(rng.integers(0, 4, m, dtype=np.uint8)))
        ex = np.array([tuple(fmpm.exact_search(idx, p)[:2]) for p in pats], dtype=np.int64)
        # inexact: z in 0..2, short patterns
        ipats, iz, irow, ik, il, idf, hits = [], [], [0], [], [], [], []
        for _ in range(60):
            m = int(rng.integers(1, 13))
            z = int(rng.integers(0, 3))
            if rng.random() < 0.6 and m <= n:
                s = int(rng.integers(0, n - m + 1))
                p = list(text[s:s + m])
                for _ in range(int(rng.integers(0, 2))):
                    j = int(rng.integers(0, m))
                    p[j] = "ACGT"[int(rng.integers(0, 4))]
                p = "".join(p)
            else:
                p = text_of(rng.integers(0, 4, m, dtype=np.uint8))
            res = fmpm.inexact_search(idx, p, z)
            ipats.append(p)
            iz.append(z)
            for r in res:
                ik.append(r.interval.k)
                il.append(r.interval.l)
                idf.append(r.diffs_used)
            irow.append(len(ik))
            h, _ = fmpm.collect_hits(idx, res, len(p))
            hits.append([(x.global_pos, x.diffs) for x in h])
        sa = fmpm.build_suffix_array(text)
        psi = [fmpm.psi_inverse_fused(idx, i) for i in range(n + 1)]
        out[f"{n}_{seed}"] = {
            "n": n, "seed": seed, "fmi_sha256": sha(fmi_bytes(idx)),
            "occ_low": low.tolist(), "occ_high": high.tolist(), "occ": occ.tolist(),
            "exact_patterns": pats, "exact_kl": ex.tolist(),
            "inexact_patterns": ipats, "inexact_z": iz, "inexact_row": irow,
            "inexact_k": ik, "inexact_l": il, "inexact_diffs": idf, "hits": hits,
            "sa": list(sa),
            "psi": [[-1, -1] if v is None else list(v) for v in psi],
            "locate": [fmpm.locate_row(idx, i) for i in range(n + 1)],
        }
    (HERE / "small_cases.json").write_text(json.dumps(out, separators=(",", ":")))
    print("small: wrote", len(out), "cases")


def gen_config0():
    wl = workloads.config0()
    t0 = time.time()
    idx = fmpm.build_index(text_of(wl.text))
    t1 = time.time()
    pats = ["".join(SYM[p]) for p in wl.patterns]
    kl = np.array([tuple(fmpm.exact_search(idx, p)[:2]) for p in pats], dtype=np.int64)
    t2 = time.time()
    np.savez_compressed(HERE / "config0_exact.npz", kl=kl.astype(np.int32))
    meta = {"fmi_sha256": sha(fmi_bytes(idx)), "text_sha256": sha(wl.text),
            "patterns_sha256": sha(wl.patterns), "kl_sha256": sha(kl.astype(np.int64)),
            "build_s": t1 - t0, "search_s": t2 - t1}
    (HERE / "config0_meta.json").write_text(json.dumps(meta, indent=1))
    print("config0:", meta)


_IDX = None


def _occ_chunk(args):
    low, high = args
    out = np.empty((low.size, 8), dtype=np.uint32)
    for i in range(low.size):
        p = fmpm.occ_pair_all(_IDX, int(low[i]), int(high[i]))
        out[i, :4] = p.at_low
        out[i, 4:] = p.at_high
    return out


def gen_config1():
    global _IDX
    wl = workloads.config1()
    t0 = time.time()
    _IDX = fmpm.build_index(text_of(wl.text))
    t1 = time.time()
    fmi = fmi_bytes(_IDX)
    low, high = wl.pairs[:, 0], wl.pairs[:, 1]
    chunks = [(low[i:i + 65536], high[i:i + 65536]) for i in range(0, low.size, 65536)]
    with mp.get_context("fork").Pool(len(os.sched_getaffinity(0))) as pool:
        parts = pool.map(_occ_chunk, chunks)
    out = np.concatenate(parts)
    t2 = time.time()
    np.savez_compressed(HERE / "config1_head.npz", occ=out[:4096])
    meta = {"fmi_sha256": sha(fmi), "pairs_sha256": sha(wl.pairs), "occ_sha256": sha(out),
            "n_pairs": int(low.size), "build_s": t1 - t0, "occ_s": t2 - t1}
    (HERE / "config1_meta.json").write_text(json.dumps(meta, indent=1))
    print("config1:", meta)


def gen_cli():
    """The reference CLI on a 3-record FASTA: match TSV/stderr at z = 0, 1, 2, --max-hits, bench checksum."""
    import contextlib

    from fmpm.cli import main as ref_main

    out = HERE / "cli"
    out.mkdir(exist_ok=True)
    rng = np.random.Generator(np.random.PCG64(777))
    recs = [("chr1", 1500), ("chr2", 900), ("chrM", 400)]
    texts = {name: text_of(rng.integers(0, 4, n, dtype=np.uint8)) for name, n in recs}
    with open(out / "ref.fa", "w") as fh:
        for name, _ in recs:
            seq = texts[name]
            fh.write(f">{name} synthetic\n")
            for i in range(0, len(seq), 70):
                fh.write(seq[i:i + 70] + "\n")
    whole = "".join(texts[n] for n, _ in recs)
    pats = []
    for _ in range(60):
        m = int(rng.integers(4, 25))
        s = int(rng.integers(0, len(whole) - m))
        p = whole[s:s + m]
        r = rng.random()
        if r < 0.3:
            j = int(rng.integers(0, m))
            p = p[:j] + "ACGT"[(("ACGT".index(p[j])) + 1) % 4] + p[j + 1:]
        elif r < 0.4:
            p = p.lower()
        pats.append(p)
    pats += ["ACNGT", "AC", "TTTTTTTTTTTTTTTTTTTT", whole[1495:1505]]  # degenerate, frequent, absent, junction
    (out / "patterns.txt").write_text("\n".join(pats) + "\n")
    fmi = out / "ref.fmi"

    def run(args, name):
        so, se = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            code = ref_main(args)
        (out / f"{name}.out").write_text(so.getvalue())
        (out / f"{name}.err").write_text(se.getvalue())
        return code

    assert run(["index", str(out / "ref.fa"), "-o", str(fmi)], "index") == 0
    (out / "ref.fmi.sha256").write_text(sha(fmi.read_bytes()))
    fmi_bytes = fmi.read_bytes()
    for z in (0, 1, 2):
        assert run(["match", str(fmi), "-f", str(out / "patterns.txt"), "-z", str(z)], f"match_z{z}") == 0
    assert run(["match", str(fmi), "-f", str(out / "patterns.txt"), "-z", "1", "--max-hits", "2"], "match_max2") == 0
    assert run(["bench", str(fmi), "--iters", "30", "--seed", "3", "--kernels", "bytelut"], "bench") == 0
    fmi.unlink()  # the tests rebuild it with our own index command
    print("cli: fixtures written", len(fmi_bytes), "byte index")


class _LazyBuckets:
    """numpy-backed stand-in for FmIndex.buckets so the UNCHANGED reference query
    code runs on indexes it cannot build itself."""

    def __init__(self, records):
        self.rec = records
        self.base = records[:, :32].view("<u8")

    def __len__(self):
        return self.rec.shape[0]

    def __getitem__(self, j):
        return fmpm.index.OccBucket(base=tuple(int(x) for x in self.base[j]), chars=self.rec[j, 32:].tobytes())


def _ref_index(ours):
    """fmpm.FmIndex over our native build (byte-identical .fmi semantics)."""
    return fmpm.FmIndex(n=ours.n, c=tuple(ours.c), buckets=_LazyBuckets(ours.bucket_records),
                        sentinel_row=ours.sentinel_row, sa_samples=tuple(int(x) for x in ours.sa_samples[:1]),
                        records=tuple(fmpm.RecordSpan(r.name, r.start, r.length) for r in ours.records))


def gen_scale():
    """Reference outputs on deterministic subsamples of the genome-scale configs."""
    from paper_1811_06127_b200 import build_index

    out = {}
    # config 4 and 1-H share the 1 Gbp text (seed 5)
    t0 = time.time()
    wl4 = workloads.config4(count=1 << 14)
    idx = build_index(wl4.text, builder="host")
    ref = _ref_index(idx)
    print(f"1 Gbp host build {time.time() - t0:.0f}s", flush=True)
    seeds = workloads.unpack_patterns(wl4.packed, 20)
    kl = np.array([tuple(fmpm.exact_search(ref, text_of(p))[:2]) for p in seeds], dtype=np.int64)
    out["config4_first16k_kl"] = kl.tolist()
    wl1h = workloads.config1h(count=1 << 12)
    occ = np.array([tuple(p.at_low) + tuple(p.at_high) for p in
                    (fmpm.occ_pair_all(ref, int(a), int(b)) for a, b in wl1h.pairs)], dtype=np.int64)
    out["config1h_first4k_occ"] = occ.tolist()
    del idx, ref
    # config 2: the first 2000 seeds of the full 1M-read set, z = 1
    wl2 = workloads.config2()
    idx = build_index(wl2.text, builder="host")
    ref = _ref_index(idx)
    res = []
    for p in wl2.patterns[:2000]:
        res.append([(m.interval.k, m.interval.l, m.diffs_used) for m in fmpm.inexact_search(ref, text_of(p), 1)])
    out["config2_first2k_z1"] = res
    (HERE / "scale_cases.json").write_text(json.dumps(out, separators=(",", ":")))
    print("scale: wrote", {k: len(v) for k, v in out.items()}, flush=True)


def gen_buckets():
    """Reference bucket kernels (kernels.py:125-358) on seeded random buckets:
    every count_bucket_* / all4 / mask_bucket answer and the nibble trace."""
    from fmpm import kernels as K

    rng = np.random.Generator(np.random.PCG64(4242))
    n = 3000
    blocks = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    blocks[:64] = 0                      # all-A buckets
    blocks[64:128] = 0xFF                # all-T buckets
    prefix = rng.integers(0, 129, n)
    prefix[:129] = np.arange(129)        # every prefix length
    symbol = rng.integers(0, 4, n)
    counts = np.zeros((n, 4), dtype=np.int64)
    all4 = np.zeros((n, 4), dtype=np.int64)
    masked = np.zeros((n, 32), dtype=np.uint8)
    trace = np.zeros((n, 15), dtype=np.uint64)
    for i in range(n):
        b, pl, sy = blocks[i].tobytes(), int(prefix[i]), int(symbol[i])
        counts[i] = [K.count_bucket_scalar(b, pl, sy), K.count_bucket_bytelut(b, pl, sy),
                     K.count_bucket_nibble(b, pl, sy), K.count_bucket_simd(b, pl, sy)]
        all4[i] = K.count_bucket_all4(b, pl)
        masked[i] = np.frombuffer(K.mask_bucket(b, pl), dtype=np.uint8)
        tr = K.KernelTrace()
        K.count_bucket_nibble(b, pl, sy, trace=tr)
        trace[i, 0:4] = tr.masked_words
        trace[i, 4:8] = tr.lookup_lo_words
        trace[i, 8:12] = tr.lookup_hi_words
        trace[i, 12] = sum(int(v) << (16 * g) for g, v in enumerate(tr.group_sads))
        trace[i, 13] = tr.sad_total | (tr.raw_count << 32)
        trace[i, 14] = tr.count
    np.savez_compressed(HERE / "buckets.npz", blocks=blocks, prefix=prefix, symbol=symbol, counts=counts,
                        all4=all4, masked=masked, trace=trace, tables_lo=np.frombuffer(K.TABLES.lo, np.uint8),
                        tables_hi=np.frombuffer(K.TABLES.hi, np.uint8))
    print("buckets: wrote", n, "cases")


class _LazySamples:
    def __init__(self, samples):
        self.s = samples

    def __len__(self):
        return self.s.size

    def __getitem__(self, j):
        return int(self.s[j])


def _ref_index_full(ours):
    """As _ref_index, with every SA sample (locate / hits)."""
    return fmpm.FmIndex(n=ours.n, c=tuple(ours.c), buckets=_LazyBuckets(ours.bucket_records),
                        sentinel_row=ours.sentinel_row, sa_samples=_LazySamples(ours.sa_samples),
                        records=tuple(fmpm.RecordSpan(r.name, r.start, r.length) for r in ours.records))


C3_READS = 8192  # config3(n_reads=C3_READS): 114,688 seeds; the tests regenerate the same call
HIT_ROWS_CAP = 2000  # hit lists are recorded for seeds whose intervals hold at most this many rows


def _hits_of(ref, matches, m):
    rows = sum(max(0, x.interval.l - x.interval.k + 1) for x in matches)
    if rows > HIT_ROWS_CAP:
        return None
    h, _ = fmpm.collect_hits(ref, matches, m)
    return [(int(x.global_pos), int(x.diffs)) for x in h]


def gen_scale3():
    """Config 3 (3.1 Gbp, rows > 2^31): the reference's exact and z = 1 results
    and hit lists on the first 2,048 seeds, through the lazy-bucket view."""
    from paper_1811_06127_b200 import build_index

    t0 = time.time()
    wl = workloads.config3(n_reads=C3_READS)
    print(f"config3 text {time.time() - t0:.0f}s", flush=True)
    idx = build_index(wl.text, builder="host")
    print(f"3.1 Gbp host build {time.time() - t0:.0f}s", flush=True)
    ref = _ref_index_full(idx)
    seeds = workloads.unpack_patterns(wl.packed[:2048], wl.meta["m"])
    ex, z1, hx, h1 = [], [], [], []
    for p in seeds:
        t = text_of(p)
        iv = fmpm.exact_search(ref, t)
        ex.append((iv.k, iv.l))
        hx.append(_hits_of(ref, [] if iv.is_empty else [fmpm.MatchResult(iv, 0)], len(t)))
        res = fmpm.inexact_search(ref, t, 1)
        z1.append([(m.interval.k, m.interval.l, m.diffs_used) for m in res])
        h1.append(_hits_of(ref, res, len(t)))
    out = {"n": int(idx.n), "text_sha256_head": sha(wl.text[:1 << 20]), "packed_sha256": sha(wl.packed[:2048]),
           "exact": ex, "z1": z1, "exact_hits": hx, "z1_hits": h1, "hit_rows_cap": HIT_ROWS_CAP,
           "fmi_meta": {"c": [int(x) for x in idx.c], "sentinel_row": int(idx.sentinel_row)}}
    (HERE / "scale3_cases.json").write_text(json.dumps(out, separators=(",", ":")))
    print(f"scale3: wrote {len(ex)} seeds in {time.time() - t0:.0f}s", flush=True)


def gen_hits():
    """Reference hit lists (collect_hits, search.py:245-267) on subsamples of
    configs 0 (exact), 2 (z = 1) and 4 (exact)."""
    from paper_1811_06127_b200 import build_index

    out = {}
    wl0 = workloads.config0()
    ref = _ref_index_full(build_index(wl0.text, builder="host"))
    out["config0_first1k_exact_hits"] = [
        _hits_of(ref, [fmpm.MatchResult(iv, 0)] if not iv.is_empty else [], len(p))
        for iv, p in ((fmpm.exact_search(ref, text_of(p)), p) for p in wl0.patterns[:1000])]
    wl2 = workloads.config2()
    ref = _ref_index_full(build_index(wl2.text, builder="host"))
    out["config2_first500_z1_hits"] = [_hits_of(ref, fmpm.inexact_search(ref, text_of(p), 1), len(p))
                                       for p in wl2.patterns[:500]]
    wl4 = workloads.config4(count=1 << 11)
    ref = _ref_index_full(build_index(wl4.text, builder="host"))
    seeds = workloads.unpack_patterns(wl4.packed, 20)
    out["config4_first2k_exact_hits"] = [
        _hits_of(ref, [fmpm.MatchResult(iv, 0)] if not iv.is_empty else [], 20)
        for iv in (fmpm.exact_search(ref, text_of(p)) for p in seeds)]
    (HERE / "hits_cases.json").write_text(json.dumps(out, separators=(",", ":")))
    print("hits: wrote", {k: len(v) for k, v in out.items()}, flush=True)


if __name__ == "__main__":
    for what in sys.argv[1:]:
        {"small": gen_small, "config0": gen_config0, "config1": gen_config1, "cli": gen_cli,
         "scale": gen_scale, "buckets": gen_buckets, "scale3": gen_scale3, "hits": gen_hits}[what]()
