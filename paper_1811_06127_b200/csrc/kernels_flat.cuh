// Flat z = 1 engine for the bounded-difference search (search.py:97-159):
// the one-edit neighbourhood of each pattern enumerated candidate by
// candidate, one WARP per pattern.  Part of libfmgpu.so (sm_100a); included
// once by fmgpu.cu after kernels_inexact.cuh.
//
// For z = 1 the reference's DFS reports (interval(S), diffs) for every string
// S within one edit of W that occurs in the text — W itself (diffs 0), a
// substitution or deletion at i in [0, m-1], an insertion after W[i], i in
// [0, m-1] (never before W[0]) — equal intervals keeping the smallest diffs;
// the visiting order is free (kernels_bidir.cuh).  When the
// pattern is only a few characters longer than the deepest k-mer table level
// (config 3: m = 19 against level 16), walking a tree shares almost nothing:
// every candidate string is ONE gather of its last min(L, kmax) characters
// away from a nearly final answer, and the gathers of different candidates
// are independent.  So instead of a per-thread DFS (8 of 32 lanes active,
// ~1 request in flight per thread) a warp takes a pattern, its lanes take the
// 8m + 1 candidates (8 per position: 4 insertions, 3 substitutions, 1
// deletion; plus W), each lane issues all its gathers back to back, and the
// candidates still alive (about half at level 16 of a 3.1 Gbp text) are
// compacted through shared memory and extended level by level — every lane
// active at every level — with one-symbol Occ steps on the index lines.
// Results are collected, sorted by (k, l) and deduplicated in shared memory;
// one atomic per pattern reserves the output rows.  No reverse index, no
// per-thread hash table, no merge pass.
//
// Pruning (result-preserving, same bound as the DFS engines): dbits marks the
// right ends of disjoint absent segments of W (k_dbound).  Two segments: no
// string within one edit occurs.  A substitution / deletion at i keeps
// W[0..i-1] verbatim, an insertion after W[i] keeps W[0..i]: a marked segment
// inside that prefix rules the candidate out.  Duplicate spellings are
// enumerated once: inserting W[i] after W[i] (i >= 1) equals inserting it
// after W[i-1]; deleting W[i] equals deleting W[i-1] when they are equal.
#pragma once

#include <cstdint>

#include "kernels_inexact.cuh"
#include "occ_device.cuh"

namespace fmg {

__device__ __forceinline__ uint64_t shl64(uint64_t x, uint32_t n) {  // PTX clamps n >= 64 to 0
  uint64_t r;
  asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(n));
  return r;
}
__device__ __forceinline__ uint64_t shr64(uint64_t x, uint32_t n) {
  uint64_t r;
  asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(n));
  return r;
}

// one table entry, no reuse expected: 64-byte DRAM fetch, no L1 allocation
__device__ __forceinline__ uint2 ld_table_entry(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::64B.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// ---- neighbourhood presence filter ----------------------------------------
// Almost every candidate is absent from the text, and finding that out costs
// a table gather plus the backward steps of the ones a 16-mer cannot rule out
// (half of them at 3.1 Gbp).  The filter answers "does this B-mer occur in
// the text" (B = table level + 2: 4^18 bits = 8.6 GB) with one bit, and it is
// stored NO times, each copy with another group of G window positions as the
// LOW digits of the bit index: the candidates that differ from each other
// only inside one group (all substitutions at G neighbouring positions, the
// four insertions at one position) then read bits of ONE 32-byte sector (G =
// 4: 256 bits), so a warp's probes of such a group are one DRAM request
// instead of one per candidate.  A candidate of length L >= B is probed
// through a B-character window that holds its edit; a clear bit ends it (for
// L == B the bit is the exact answer).  Built from the level-kx k-mer table by
// a depth-(B - kx) traversal (k_flat_filter_build): "occurs" = "backward
// search leaves a non-empty interval", the engines' own notion.
struct FlatFilter {
  const uint32_t* bits = nullptr;  // NO bitmaps of 4^B bits
  uint32_t B = 0, G = 0, NO = 0;
  uint32_t rcpG = 0;  // ceil(2^32 / G), G >= 2: x / G = umulhi(x, rcpG) for the small x used here
};

// Bit index of window w (B characters, character t in bits 2t..2t+1) in copy
// o: the group's G digits first, the other digits in order above them.
__device__ __forceinline__ uint64_t filter_key(const FlatFilter& f, uint64_t w, uint32_t o) {
  const uint32_t gs = min(o * f.G, f.B - f.G);
  const uint64_t mg = shl64(1ull, 2u * f.G) - 1ull;
  const uint64_t below = w & (shl64(1ull, 2u * gs) - 1ull);
  const uint64_t above = shl64(shr64(w, 2u * (gs + f.G)), 2u * (gs + f.G));
  return (shr64(w, 2u * gs) & mg) | shl64(below, 2u * f.G) | above;
}

__device__ __forceinline__ uint64_t filter_word(const FlatFilter& f, uint64_t key, uint32_t o) {
  return (uint64_t(o) << (2u * f.B - 5u)) + (key >> 5);
}

// Window and copy a candidate is probed through: e = position of the edited
// character in S (substitution: i; insertion after W[i]: i + 1; deletion of
// W[i]: the character that followed it, or the last one), the first window
// when it holds e, else the last.
__device__ __forceinline__ uint64_t filter_probe_addr(const FlatFilter& f, uint32_t c, int m, uint64_t S, int L,
                                                      uint32_t& bit) {
  const uint32_t i = c >> 3, s = c & 7u;
  const uint32_t e = c >= uint32_t(8 * m) ? 0u : s < 4u ? i + 1u : s < 7u ? i : min(i, uint32_t(L) - 1u);
  const uint32_t ws = e < f.B ? 0u : uint32_t(L) - f.B;
  const uint64_t w = shr64(S, 2u * ws) & (shl64(1ull, 2u * f.B) - 1ull);
  const uint32_t o = min(__umulhi(e - ws, f.rcpG), f.NO - 1u);
  const uint64_t key = filter_key(f, w, o);
  bit = uint32_t(key) & 31u;
  return filter_word(f, key, o);
}

__device__ __forceinline__ uint32_t ld_filter_word(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Candidate c of pattern pw (m characters, character t in bits 2t..2t+1):
// c = 8i + s, s = 0..3 insertion of s after W[i], s = 4..6 substitution of
// W[i] by (W[i] + s - 3) & 3, s = 7 deletion of W[i]; c = 8m is W itself.
// Returns the string S (L characters, same packing) and whether it has to be
// searched at all.
//
// Branch-free on purpose: the lanes of a warp hold all three kinds of edit,
// and a branch per kind made the warp run the probe code after it three times
// over (ncu: 1,200 of 2,500 warp instructions per pattern).  Every candidate
// is one splice: the first a characters of W, `put` inserted characters (b),
// then W from position i + 1 on.
__device__ __forceinline__ bool flat_candidate(uint64_t pw, int m, uint64_t db, uint32_t c, uint64_t& S, int& L) {
  const uint32_t m8 = 8u * uint32_t(m);
  const bool is_w = c >= m8;  // W itself (c == 8m), or padding past it
  const uint32_t i = is_w ? 0u : c >> 3, s = c & 7u;
  const bool ins = s < 4u, del = s == 7u;
  const uint32_t wi = uint32_t(shr64(pw, 2u * i)) & 3u;
  const uint32_t wprev = uint32_t(shr64(pw, 2u * i - 2u)) & 3u;  // W[i-1] (i >= 1; unused otherwise)
  const uint32_t b = ins ? s : (wi + s - 3u) & 3u;               // inserted / substituted character
  const uint32_t a = i + (ins ? 1u : 0u);                         // characters of W kept below the edit
  const uint32_t put = del ? 0u : 1u;
  const uint64_t low = pw & (shl64(1ull, 2u * a) - 1ull);
  const uint64_t mid = shl64(uint64_t(del ? 0u : b), 2u * a);
  const uint64_t high = shl64(shr64(pw, 2u * i + 2u), 2u * (a + put));  // W[i+1..]
  const bool prev_ok = (db & (shl64(1ull, i) - 1ull)) == 0ull;   // no absent segment inside W[0..i-1]
  const bool cur_ok = (db & (shl64(2ull, i) - 1ull)) == 0ull;    // ... inside W[0..i]
  const bool ok_ins = cur_ok && (s != wi || i == 0u);
  const bool ok_del = prev_ok && !(i >= 1u && wi == wprev);
  const bool ok = ins ? ok_ins : del ? ok_del : prev_ok;
  S = is_w ? pw : (low | mid | high);
  L = m + (is_w ? 0 : (ins ? 1 : 0) - (del ? 1 : 0));
  return is_w ? (c == m8 && db == 0ull) : ok;
}

// Raw line data of one backward step at (k-1, l): the high line always, the
// low line only when it is a different one (W = 2: predicated, no request).
template <int W>
struct StepLines {
  uint32_t bh[4], bl[4];
  uint64_t wh[W], wl[W];
  uint32_t jh, jl;
};

template <int W>
__device__ __forceinline__ void step_load(const IndexView& ix, bool go, uint32_t k, uint32_t l, StepLines<W>& sl) {
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint32_t low = k - 1u;
  sl.jh = line_of<W>(l);
  sl.jl = line_of<W>(low);
  if constexpr (W == 2) {
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    ld256_pred(go, ix.lines + size_t(sl.jh) * LineTraits<2>::kBytes, a0, a1, a2, a3);
    ld256_pred(go && sl.jl != sl.jh, ix.lines + size_t(sl.jl) * LineTraits<2>::kBytes, b0, b1, b2, b3);
    const bool same = sl.jl == sl.jh;
    sl.bh[0] = uint32_t(a0), sl.bh[1] = uint32_t(a0 >> 32), sl.bh[2] = uint32_t(a1), sl.bh[3] = uint32_t(a1 >> 32);
    sl.wh[0] = a2, sl.wh[1] = a3;
    sl.bl[0] = same ? sl.bh[0] : uint32_t(b0);
    sl.bl[1] = same ? sl.bh[1] : uint32_t(b0 >> 32);
    sl.bl[2] = same ? sl.bh[2] : uint32_t(b1);
    sl.bl[3] = same ? sl.bh[3] : uint32_t(b1 >> 32);
    sl.wl[0] = same ? a2 : b2;
    sl.wl[1] = same ? a3 : b3;
  } else {
    if (go) {
      load_line<W, 0>(ix, sl.jh, l - sl.jh * kC, sl.bh, sl.wh);
      load_line<W, 0>(ix, sl.jl, low - sl.jl * kC, sl.bl, sl.wl);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) sl.bh[t] = sl.bl[t] = 0u;
#pragma unroll
      for (int t = 0; t < W; ++t) sl.wh[t] = sl.wl[t] = 0ull;
    }
  }
}

template <int W>
__device__ __forceinline__ void step_finish(const IndexView& ix, const StepLines<W>& sl, uint32_t sym, uint32_t& k,
                                            uint32_t& l) {
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint32_t low = k - 1u;
  const uint32_t cs = c_of(ix, sym);
  const uint32_t k2 = cs + occ1_from_line<W>(ix, sl.bl, sl.wl, low, low - sl.jl * kC, sym) + 1u;
  const uint32_t l2 = cs + occ1_from_line<W>(ix, sl.bh, sl.wh, l, l - sl.jh * kC, sym);
  k = k2;
  l = l2;
}

// NR = rounds of 32 candidates a lane takes (32 NR >= 8m + 1).  Shared
// memory per warp, cap = 32 NR slots each: the candidates that passed the
// filter (cq), the continuation queue (k, l, candidate | next position << 16,
// and the candidate's first 16 characters: the ones still to prepend), the
// results (k, l) and one flag word per 32 results.  Only W itself carries
// diffs 0, so the diffs of a result are "is it the exact one" (its index is
// kept in a register).
//
// Instruction budget (ncu, config 3): the first form of this kernel spent
// 3,800 warp instructions per pattern, a quarter of them rebuilding the
// candidate string three times per candidate, and was issue-bound once the
// filter had removed most memory requests.  Now a candidate string is built
// once for its probe, and again only if it survives (7 %); the continuation
// queue carries the characters still needed; results are deduplicated with
// one match instruction when there are at most 32.
#ifndef FMG_FLAT_MINB
#define FMG_FLAT_MINB 8  // resident 128-thread blocks per SM the register budget is sized for
#endif

template <int NR>
struct FlatSmem {
  static constexpr uint32_t cap = 32u * NR;
  static constexpr uint32_t words_per_warp = 7u * cap + NR;
};

template <int W, int NR>
__global__ void __launch_bounds__(128, FMG_FLAT_MINB) k_z1_flat(IndexView ix, PrefixTable tf, const uint2* __restrict__ tx,
                                                 uint32_t kx, CodePatterns cp, const uint32_t* __restrict__ list,
                                                 uint64_t count, InexactOut out, FlatFilter flt) {
  extern __shared__ __align__(16) uint32_t flat_smem[];
  constexpr uint32_t cap = FlatSmem<NR>::cap;
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  uint32_t* kq = flat_smem + wib * FlatSmem<NR>::words_per_warp;
  uint32_t* lq = kq + cap;
  uint32_t* xq = lq + cap;
  uint32_t* sq = xq + cap;
  uint32_t* cq = sq + cap;
  uint32_t* kr = cq + cap;
  uint32_t* lr = kr + cap;
  uint32_t* repw = lr + cap;
  const uint32_t K = tf.k, kmax = tx ? kx : K;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint64_t work = 0;

  // the next pattern is claimed and loaded while the current one is searched
  uint64_t nq_id = 0, npw = 0, ndb = 0;
  int nm = 0;
  bool nvalid = false;
  auto prefetch = [&]() {
    unsigned long long slot = 0;
    if (lane == 0u) slot = atomicAdd(out.next, 1ull);
    slot = __shfl_sync(0xFFFFFFFFu, slot, 0);
    nvalid = slot < count;
    if (!nvalid) return;
    nq_id = list ? list[slot] : slot;
    if (cp.packed1) {
      nm = int(cp.fixed_m);
      npw = cp.packed1[nq_id];
    } else {
      nm = int(cp.offsets[nq_id + 1] - cp.offsets[nq_id]);
      npw = cp.packed[nq_id].x;
    }
    ndb = cp.dbits[nq_id];
  };
  prefetch();

  while (nvalid) {
    const uint64_t q = nq_id;
    const int m = nm;
    const uint64_t pw = npw & (shl64(1ull, 2u * uint32_t(m)) - 1ull);  // m <= 31
    const uint64_t db = ndb;
    prefetch();
    const uint32_t NC = 8u * uint32_t(m) + 1u;
    uint32_t nres = 0;
    uint32_t exact_idx = 0xFFFFFFFFu;  // result index of W itself
    // a finished candidate joins the results
    auto add_results = [&](bool done, uint32_t c, uint32_t k, uint32_t l) {
      const uint32_t bd = __ballot_sync(0xFFFFFFFFu, done);
      if (bd == 0u) return;
      const uint32_t idx = nres + __popc(bd & lt_mask);
      if (done) {
        kr[idx] = k;
        lr[idx] = l;
      }
      const uint32_t be = __ballot_sync(0xFFFFFFFFu, done && c == NC - 1u);
      if (be) exact_idx = __shfl_sync(0xFFFFFFFFu, idx, __ffs(be) - 1);
      nres += __popc(bd);
    };

    if (__popcll(db) <= 1) {
      // ---- the candidates worth searching: every probe issued, then read ----
      uint32_t fw[NR];
      uint32_t vmask = 0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const uint32_t c = uint32_t(r) * 32u + lane;
        uint64_t S;
        int L;
        fw[r] = 1u;
        if (c < NC && flat_candidate(pw, m, db, c, S, L)) {
          vmask |= 1u << r;
          if (flt.bits && uint32_t(L) >= flt.B) {
            uint32_t bit;
            const uint64_t a = filter_probe_addr(flt, c, m, S, L, bit);
            fw[r] = ld_filter_word(flt.bits + a) >> bit;
            work += 1ull;  // one sector, no Occ step
          }
        }
      }
      uint32_t nc = 0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const bool pass = ((vmask >> r) & 1u) && (fw[r] & 1u);
        const uint32_t bp = __ballot_sync(0xFFFFFFFFu, pass);
        if (pass) cq[nc + __popc(bp & lt_mask)] = uint32_t(r) * 32u + lane;
        nc += __popc(bp);
      }
      __syncwarp();
      // ---- their table gathers (two chunks of 32 in flight), finished ones
      // to the results, the others to the continuation queue ----
      uint32_t nq = 0;
      for (uint32_t base = 0; base < nc; base += 64u) {
        uint2 e[2];
        uint32_t cc[2], s32[2];
        int pos[2];
        bool go[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t j = base + 32u * u + lane;
          go[u] = j < nc;
          cc[u] = 0u, s32[u] = 0u, pos[u] = -1;
          e[u] = make_uint2(1u, 0u);
          if (u == 1 && base + 32u >= nc) continue;  // warp-uniform
          if (go[u]) {
            cc[u] = cq[j];
            uint64_t S;
            int L;
            flat_candidate(pw, m, db, cc[u], S, L);
            s32[u] = uint32_t(S);
            e[u] = make_uint2(0u, ix.n);  // the empty string (a deletion from m = 1)
            const uint32_t d = min(uint32_t(L), kmax);
            pos[u] = L - int(d) - 1;  // next character to prepend
            if (L > 0) {
              const uint32_t key = uint32_t(S >> (2u * (uint32_t(L) - d))) & uint32_t(shl64(1ull, 2u * d) - 1ull);
              e[u] = ld_table_entry(d > K ? tx + key : tf.base + PrefixTable::off(d) + key);
              work += work_unit(1u);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && base + 32u >= nc) continue;
          const bool alive = go[u] && e[u].x <= e[u].y;
          const bool cont = alive && pos[u] >= 0;
          add_results(alive && pos[u] < 0, cc[u], e[u].x, e[u].y);
          const uint32_t bc = __ballot_sync(0xFFFFFFFFu, cont);
          if (cont) {
            const uint32_t slot = nq + __popc(bc & lt_mask);
            kq[slot] = e[u].x;
            lq[slot] = e[u].y;
            xq[slot] = cc[u] | (uint32_t(pos[u]) << 16);
            sq[slot] = s32[u];
          }
          nq += __popc(bc);
        }
      }
      __syncwarp();
      // ---- level by level: one backward step for every queued candidate ----
      while (nq > 0u) {
        uint32_t nnew = 0;
        for (uint32_t base = 0; base < nq; base += 64u) {
          const bool two = base + 32u < nq;  // warp-uniform
          uint32_t k[2], l[2], x[2], sv[2];
          bool go[2];
          StepLines<W> sl[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint32_t j = base + 32u * u + lane;
            go[u] = j < nq;
            k[u] = go[u] ? kq[j] : 1u;
            l[u] = go[u] ? lq[j] : 0u;
            x[u] = go[u] ? xq[j] : 0u;
            sv[u] = go[u] ? sq[j] : 0u;
          }
          __syncwarp();  // the chunk is in registers before its slots are reused (nnew <= base + 64)
          step_load<W>(ix, go[0], k[0], l[0], sl[0]);
          if (two) step_load<W>(ix, go[1], k[1], l[1], sl[1]);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) continue;
            const uint32_t c = x[u] & 0xFFFFu, pos = x[u] >> 16;
            uint32_t sym = (sv[u] >> (2u * (pos & 15u))) & 3u;
            if (pos >= 16u) {  // beyond the 16 characters the queue carries (never in production shapes)
              uint64_t S;
              int L;
              flat_candidate(pw, m, db, c, S, L);
              sym = uint32_t(S >> (2u * pos)) & 3u;
            }
            if (go[u]) work += work_unit(sl[u].jl != sl[u].jh ? 2u : 1u);
            step_finish<W>(ix, sl[u], sym, k[u], l[u]);
            const bool alive = go[u] && k[u] <= l[u];
            const bool cont = alive && pos != 0u;
            add_results(alive && pos == 0u, c, k[u], l[u]);
            const uint32_t bc = __ballot_sync(0xFFFFFFFFu, cont);
            if (cont) {
              const uint32_t slot = nnew + __popc(bc & lt_mask);
              kq[slot] = k[u];
              lq[slot] = l[u];
              xq[slot] = c | ((pos - 1u) << 16);
              sq[slot] = sv[u];
            }
            nnew += __popc(bc);
          }
        }
        nq = nnew;
        __syncwarp();
      }
    }

    // ---- results: representatives (first of each interval, W itself before
    // the others), their rank among the distinct intervals, one reservation,
    // ordered write ----
    __syncwarp();
    if (nres <= 32u) {
      // one result per lane: equal intervals found by one match instruction
      const bool have = lane < nres;
      const uint32_t mk = have ? kr[lane] : 0xFFFFFFFFu, ml = have ? lr[lane] : lane;
      const unsigned long long key = (uint64_t(mk) << 32) | ml;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
      const uint32_t be = exact_idx < 32u ? (1u << exact_idx) : 0u;
      const bool with_exact = (peers & be) != 0u;
      const bool rep = have && (with_exact ? lane == exact_idx : lane == uint32_t(__ffs(peers) - 1));
      const uint32_t repmask = __ballot_sync(0xFFFFFFFFu, rep);
      const uint32_t nuniq = __popc(repmask);
      unsigned long long o = 0;
      if (lane == 0u && nuniq) o = atomicAdd(out.total, (unsigned long long)nuniq);
      o = __shfl_sync(0xFFFFFFFFu, o, 0);
      if (o + nuniq > out.cap) {  // this pass's buffer is full: retried by the next pass
        if (lane == 0u) {
          const unsigned long long f = atomicAdd(out.fail_count, 1ull);
          out.fail_list[f] = uint32_t(q);
          out.res_cnt[q] = 0u;
        }
        __syncwarp();
        continue;
      }
      uint32_t rank = 0;
      for (uint32_t rest = repmask; rest; rest &= rest - 1u) {
        const unsigned long long kj = __shfl_sync(0xFFFFFFFFu, key, __ffs(rest) - 1);
        rank += kj < key ? 1u : 0u;
      }
      if (rep) {
        out.kl[o + rank] = make_uint2(mk, ml);
        out.diffs[o + rank] = with_exact ? uint8_t(0) : uint8_t(1);
      }
      if (lane == 0u) {
        out.res_off[q] = o;
        out.res_cnt[q] = nuniq;
        out.res_pass[q] = out.pass;
      }
      __syncwarp();
      continue;
    }
    uint32_t rep_bits = 0;  // bit t: result 32 t + lane represents its interval
    uint32_t nuniq = 0;
    for (uint32_t t = 0; t * 32u < nres; ++t) {
      const uint32_t r = t * 32u + lane;
      const bool have = r < nres;
      const uint32_t mk = kr[have ? r : 0u], ml = lr[have ? r : 0u];
      const uint32_t md = r == exact_idx ? 0u : 1u;
      bool rep = have;
      for (uint32_t j = 0; j < nres; ++j) {
        const uint32_t dj = j == exact_idx ? 0u : 1u;
        if (kr[j] == mk && lr[j] == ml && (dj < md || (dj == md && j < r))) rep = false;
      }
      const uint32_t br = __ballot_sync(0xFFFFFFFFu, rep);
      if (lane == 0u) repw[t] = br;
      rep_bits |= rep ? (1u << t) : 0u;
      nuniq += __popc(br);
    }
    __syncwarp();
    unsigned long long o = 0;
    if (lane == 0u && nuniq) o = atomicAdd(out.total, (unsigned long long)nuniq);
    o = __shfl_sync(0xFFFFFFFFu, o, 0);
    if (o + nuniq > out.cap) {  // this pass's buffer is full: retried by the next pass
      if (lane == 0u) {
        const unsigned long long f = atomicAdd(out.fail_count, 1ull);
        out.fail_list[f] = uint32_t(q);
        out.res_cnt[q] = 0u;
      }
      __syncwarp();
      continue;
    }
    for (uint32_t t = 0; t * 32u < nres; ++t) {
      const uint32_t r = t * 32u + lane;
      if (r < nres && ((rep_bits >> t) & 1u)) {
        const uint32_t mk = kr[r], ml = lr[r];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < nres; ++j) {
          const uint32_t kj = kr[j], lj = lr[j];
          rank += (((repw[j >> 5] >> (j & 31u)) & 1u) && (kj < mk || (kj == mk && lj < ml))) ? 1u : 0u;
        }
        out.kl[o + rank] = make_uint2(mk, ml);
        out.diffs[o + rank] = r == exact_idx ? uint8_t(0) : uint8_t(1);
      }
    }
    if (lane == 0u) {
      out.res_off[q] = o;
      out.res_cnt[q] = nuniq;
      out.res_pass[q] = out.pass;
    }
    __syncwarp();
  }
  flush_work(out.steps, work);
}

// Filter build: entry x of the level-kx table (a present kx-mer and its
// interval) is extended D = B - kx characters to the left; every B-mer that
// still has a non-empty interval sets its bit in each of the NO copies.
template <int W, int D>
__device__ __forceinline__ void filter_expand(const IndexView& ix, const FlatFilter& f, uint32_t* bits, uint32_t k,
                                              uint32_t l, uint64_t key) {
  if constexpr (D == 0) {
    for (uint32_t o = 0; o < f.NO; ++o) {
      const uint64_t kk = filter_key(f, key, o);
      atomicOr(bits + filter_word(f, kk, o), 1u << (uint32_t(kk) & 31u));
    }
  } else {
    uint32_t lo[4], hi[4];
    occ_step<W, 0>(ix, k, l, lo, hi);
#pragma unroll 1
    for (uint32_t c = 0; c < 4u; ++c) {
      const uint32_t cs = c_of(ix, c);
      const uint32_t k2 = cs + sel4(lo, c) + 1u, l2 = cs + sel4(hi, c);
      if (k2 <= l2) filter_expand<W, D - 1>(ix, f, bits, k2, l2, (key << 2) | c);
    }
  }
}

template <int W, int D>
__global__ void __launch_bounds__(256) k_flat_filter_build(IndexView ix, const uint2* __restrict__ tx, uint64_t cnt,
                                                           FlatFilter f, uint32_t* __restrict__ bits) {
  const uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= cnt) return;
  const uint2 e = tx[x];
  if (e.x > e.y) return;
  filter_expand<W, D>(ix, f, bits, e.x, e.y, x);
}

}  // namespace fmg
