// Flat z = 1 engine for the bounded-difference search (search.py:97-159):
// the one-edit neighbourhood of each pattern enumerated string by string.
// Part of libfmgpu.so (sm_100a); included once by fmgpu.cu after
// kernels_inexact.cuh.
//
// For z = 1 the reference's DFS reports (interval(S), diffs) for every string
// S within one edit of W that occurs in the text — W itself (diffs 0), a
// substitution or deletion at i in [0, m-1], an insertion after W[i], i in
// [0, m-1] (never before W[0]) — equal intervals keeping the smallest diffs;
// the visiting order is free (kernels_bidir.cuh).  When the
// pattern is only a few characters longer than the deepest k-mer table level
// (config 3: m = 19 against level 16), walking a tree shares almost nothing:
// every candidate string is ONE gather of its last min(L, kmax) characters
// away from a nearly final answer, and the candidates are independent.
//
// Three kernels, each with the thread mapping its work wants (the first form
// was one warp-per-pattern kernel: 3,800 warp instructions per pattern with
// a third of the lanes idle after the first phase, issue-bound):
//   k_flat_probe    a warp per pattern, a lane per (kind of edit, position):
//                   the lane builds its up to four candidate strings as one
//                   splice of W, asks the presence filter about each (below)
//                   and the warp appends the survivors — the candidates the
//                   text may hold — to a queue, one contiguous segment per
//                   pattern, W itself first;
//   k_flat_extend   a thread per survivor: one table gather, then one-symbol
//                   backward steps on the index lines until the string is
//                   complete or its interval empties; the interval (or
//                   "absent") goes to the survivor's own slot, so results stay
//                   grouped by pattern without a sort;
//   k_flat_collect  a warp per pattern: its segment's intervals, sorted by
//                   (k, l) and deduplicated (one match instruction when there
//                   are at most 32), written to the pass's output buffer with
//                   one reservation.
// No reverse index, no per-thread hash table, no merge pass.
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

__device__ __forceinline__ uint32_t ld_filter_word(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
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

// One candidate the text may hold: the string S (L characters, character t
// in bits 2t..2t+1) of pattern q.
struct __align__(16) FlatSurvivor {
  uint64_t S;
  uint32_t q, L;
};

// Queues of one pass: survivors, their intervals (same index; k > l =
// absent), and per pattern the segment both share.  seg_cnt bit 31: the
// segment's first entry is W itself (diffs 0).
struct FlatQueues {
  FlatSurvivor* surv;
  uint2* raw;
  unsigned long long* n_surv;
  uint64_t cap;
  uint64_t* seg_base;
  uint32_t* seg_cnt;
};

constexpr uint32_t kFlatExactBit = 0x80000000u;
constexpr uint32_t kFlatSlab = 512u;        // queue entries a warp reserves at a time (> kFlatMaxCand)
constexpr uint32_t kFlatDead = 0xFFFFFFFFu;  // FlatSurvivor::L of an unused queue entry
constexpr uint32_t kFlatMaxCand = 8u * 31u + 1u;  // candidates of the longest pattern (m <= 31)

// ---- k_flat_probe ----------------------------------------------------------
// Slot t of a pattern: t = 0 is W itself, then m substitution slots (the
// three other characters at i), m insertion slots (the four characters after
// W[i]; never W[i] itself unless i = 0), m deletion slots.  Every slot is one
// splice — the first a characters of W, a gap of `put` characters, then W
// from position i + 1 on — whose variants differ only in the gap, so a slot
// computes one filter address and its variants read bits next to each other.
// Branch-free: a warp holds every kind of slot.
// NRS = rounds of 32 slots a lane takes (32 NRS >= 3m + 1).
// kFixed: every pattern has cp.fixed_m characters (the packed entry points),
// so the slots' geometry — kind, position, window, copy, shifts — is the same
// for every pattern and is computed once per thread, outside the pattern loop.
template <int NRS, bool kFixed>
__global__ void __launch_bounds__(256) k_flat_probe(CodePatterns cp, const uint32_t* __restrict__ list, uint64_t q0,
                                                    uint64_t count, FlatFilter flt, FlatQueues fq, InexactOut out) {
  // Queue space comes in slabs of kFlatSlab entries, one per warp at a time:
  // a same-address atomic per pattern capped the kernel at ~0.6 G patterns/s,
  // and one per block and round of patterns cost 17 % of the warps' time at
  // its barriers.  What a warp leaves unused of a slab is marked dead.
  uint64_t slab_pos = 0, slab_end = 0;
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint64_t per_round = uint64_t(gridDim.x) * 8u;
  uint64_t work = 0;
  // pattern words of the next round are loaded while this one is probed
  auto load_pattern = [&](uint64_t w, uint64_t& q, int& m, uint64_t& pw, uint64_t& db) {
    q = 0, m = 0, pw = 0, db = 0;
    if (w >= count) return;
    q = list ? list[q0 + w] : q0 + w;
    if (kFixed) {
      m = int(cp.fixed_m);
      pw = cp.packed1[q];
    } else if (cp.packed1) {
      m = int(cp.fixed_m);
      pw = cp.packed1[q];
    } else {
      m = int(cp.offsets[q + 1] - cp.offsets[q]);
      pw = cp.packed[q].x;
    }
    db = cp.dbits[q];
  };
  uint64_t nq, npw, ndb;
  int nm;
  load_pattern(uint64_t(blockIdx.x) * 8u + wib, nq, nm, npw, ndb);
  for (uint64_t wb = uint64_t(blockIdx.x) * 8u; wb < count; wb += per_round) {
    const bool active = wb + wib < count;
    const uint64_t q = nq, db = ndb;
    const int m = kFixed ? int(cp.fixed_m) : nm;
    const uint64_t pw = npw & (shl64(1ull, 2u * uint32_t(m)) - 1ull);  // m <= 31
    load_pattern(wb + per_round + wib, nq, nm, npw, ndb);
    // two absent segments: nothing within one edit occurs
    const bool search = active && __popcll(db) <= 1;
    const uint32_t first_db = db ? uint32_t(__ffsll((long long)db) - 1) : 64u;
    const uint32_t um = uint32_t(m);
    uint64_t S0[NRS];
    uint32_t meta[NRS];  // survivor variants (4 bits) | a << 8 | L << 16
    uint32_t total = 0, pre[NRS];
#pragma unroll
    for (int r = 0; r < NRS; ++r) {
      const uint32_t t = uint32_t(r) * 32u + lane;
      const bool is_w = t == 0u, slot_ok = search && t <= 3u * um;
      const uint32_t u = t - 1u;
      const uint32_t ty = is_w ? 0u : (u >= um ? 1u : 0u) + (u >= 2u * um ? 1u : 0u);  // 0 sub, 1 ins, 2 del
      const uint32_t i = is_w ? 0u : u - ty * um;
      const uint32_t wi = uint32_t(shr64(pw, 2u * i)) & 3u;
      const uint32_t wprev = uint32_t(shr64(pw, 2u * i - 2u)) & 3u;  // W[i-1] (i >= 1; unused otherwise)
      const bool prev_ok = first_db >= i, cur_ok = first_db > i;
      const uint32_t others = 0xFu & ~(1u << wi);
      uint32_t vm = ty == 0u ? (prev_ok ? others : 0u)
                  : ty == 1u ? (cur_ok ? (i == 0u ? 0xFu : others) : 0u)
                             : ((prev_ok && !(i >= 1u && wi == wprev)) ? 1u : 0u);
      if (is_w) vm = db == 0ull ? 1u : 0u;
      if (!slot_ok) vm = 0u;
      const uint32_t a = is_w ? 0u : i + (ty == 1u ? 1u : 0u);
      const uint32_t put = ty == 2u ? 0u : 1u;
      const uint64_t low = pw & (shl64(1ull, 2u * a) - 1ull);
      const uint64_t high = shl64(shr64(pw, 2u * i + 2u), 2u * (a + put));
      const uint64_t s0 = is_w ? pw : (low | high);
      const uint32_t L = um + (is_w ? 0u : (ty == 1u ? 1u : 0u)) - ((!is_w && ty == 2u) ? 1u : 0u);
      uint32_t sm = vm;
      if (flt.bits && L >= flt.B && vm) {
        // the window that holds the edit: the first one when it does, else the last
        const uint32_t e = is_w ? 0u : ty == 2u ? min(a, L - 1u) : a;
        const uint32_t ws = e < flt.B ? 0u : L - flt.B;
        const uint32_t p = e - ws;
        const uint32_t o = min(__umulhi(p, flt.rcpG), flt.NO - 1u);
        const uint32_t gs = min(o * flt.G, flt.B - flt.G);
        const uint64_t key0 = filter_key(flt, shr64(s0, 2u * ws) & (shl64(1ull, 2u * flt.B) - 1ull), o);
        // variant b sets the gap digit (zero in key0, inside the copy's group,
        // below bit 2G): the word and bit of each variant by 32-bit offsets
        const uint32_t* w0 = flt.bits + filter_word(flt, key0, o);
        const uint32_t bit0 = uint32_t(key0) & 31u, sh = 2u * (p - gs);
        uint32_t got = 0;
#pragma unroll
        for (uint32_t b = 0; b < 4u; ++b) {
          const uint32_t delta = (b << sh) + bit0;  // no carry into a set bit: key0's gap digit is zero
          if ((vm >> b) & 1u) got |= ((ld_filter_word(w0 + (delta >> 5)) >> (delta & 31u)) & 1u) << b;
        }
        work += uint64_t(__popc(vm));  // one sector each, no Occ step
        sm = got;
      }
      S0[r] = s0;
      meta[r] = sm | (a << 8) | (L << 16);
      // this round's survivors: offsets within the pattern's segment
      const uint32_t cnt = uint32_t(__popc(sm));
      uint32_t prefix = 0, rt = 0;
#pragma unroll
      for (int bit = 0; bit < 3; ++bit) {
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (cnt >> bit) & 1u);
        prefix += uint32_t(__popc(bal & lt_mask)) << bit;
        rt += uint32_t(__popc(bal)) << bit;
      }
      pre[r] = total + prefix;
      total += rt;
    }
    const uint32_t has_exact = __shfl_sync(0xFFFFFFFFu, meta[0] & 1u, 0);  // slot 0 = W itself, first in the segment
    if (!active) continue;
    if (slab_pos + total > slab_end) {  // a new slab (total <= kFlatMaxCand < kFlatSlab)
      for (uint64_t t = slab_pos + lane; t < slab_end; t += 32u) fq.surv[t].L = kFlatDead;
      unsigned long long nb = 0;
      if (lane == 0u) nb = atomicAdd(fq.n_surv, (unsigned long long)kFlatSlab);
      slab_pos = __shfl_sync(0xFFFFFFFFu, nb, 0);
      slab_end = min(slab_pos + kFlatSlab, fq.cap);
      if (slab_pos > slab_end) slab_pos = slab_end;  // past the queue: every reservation fails from here on
    }
    const unsigned long long base = slab_pos;
    if (base + total > slab_end) {  // the chunk's patterns kept more candidates than it was sized for: retried
      if (lane == 0u) {
        const unsigned long long f = atomicAdd(out.fail_count, 1ull);
        out.fail_list[f] = uint32_t(q);
        out.res_cnt[q] = 0u;
        fq.seg_base[q] = 0;
        fq.seg_cnt[q] = 0xFFFFFFFFu;  // k_flat_collect skips it
      }
      continue;
    }
#pragma unroll
    for (int r = 0; r < NRS; ++r) {
      const uint32_t a = (meta[r] >> 8) & 0xFFu, L = meta[r] >> 16;
      uint64_t slot = base + pre[r];
      for (uint32_t rest = meta[r] & 0xFu; rest; rest &= rest - 1u) {  // few lanes keep anything: a short loop
        const uint32_t b = uint32_t(__ffs(rest)) - 1u;
        FlatSurvivor sv;
        sv.S = S0[r] | shl64(uint64_t(b), 2u * a);
        sv.q = uint32_t(q);
        sv.L = L;
        fq.surv[slot++] = sv;
      }
    }
    slab_pos += total;
    if (lane == 0u) {
      fq.seg_base[q] = base;
      fq.seg_cnt[q] = total | (has_exact ? kFlatExactBit : 0u);
    }
  }
  for (uint64_t t = slab_pos + lane; t < slab_end; t += 32u) fq.surv[t].L = kFlatDead;
  flush_work(out.steps, work);
}

// ---- k_flat_extend ---------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(256) k_flat_extend(IndexView ix, PrefixTable tf, const uint2* __restrict__ tx,
                                                     uint32_t kx, FlatQueues fq, unsigned long long* steps) {
  const uint64_t n = min(uint64_t(*fq.n_surv), fq.cap);
  const uint32_t K = tf.k, kmax = tx ? kx : K;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t work = 0;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
    const FlatSurvivor sv = fq.surv[t];
    const uint32_t L = sv.L;
    if (L == kFlatDead) continue;  // the unused tail of a warp's slab
    const uint32_t d = min(L, kmax);
    uint2 e = make_uint2(0u, ix.n);  // the empty string (a deletion from m = 1)
    if (L > 0u) {
      const uint32_t key = uint32_t(shr64(sv.S, 2u * (L - d))) & uint32_t(shl64(1ull, 2u * d) - 1ull);
      e = ld_table_entry(d > K ? tx + key : tf.base + PrefixTable::off(d) + key);
      work += work_unit(1u);
    }
    uint32_t k = e.x, l = e.y;
    int pos = int(L) - int(d) - 1;  // next character to prepend
    while (k <= l && pos >= 0) {
      StepLines<W> sl;
      step_load<W>(ix, true, k, l, sl);
      work += work_unit(sl.jl != sl.jh ? 2u : 1u);
      step_finish<W>(ix, sl, uint32_t(shr64(sv.S, 2u * uint32_t(pos))) & 3u, k, l);
      --pos;
    }
    fq.raw[t] = k <= l ? make_uint2(k, l) : make_uint2(1u, 0u);
  }
  flush_work(steps, work);
}

// ---- k_flat_collect --------------------------------------------------------
// Results of a pattern: representatives (first of each interval, W itself
// before the others), their rank among the distinct intervals, ordered write.
// A warp per pattern; at most 32 candidates of the pattern survived the
// filter in the common case, so each lane holds one and a match instruction
// finds the equal intervals.  Output rows: with the filter the pattern's
// survivor segment doubles as its reservation (rows *row_base + seg_base ..;
// no atomics — k_flat_advance chains the chunks' row bases);
// without one (every candidate is a survivor, few are results) one atomic
// per pattern reserves exactly the rows used.
template <bool kSegmentRows>
__global__ void __launch_bounds__(256) k_flat_collect(const uint32_t* __restrict__ list, uint64_t q0, uint64_t count,
                                                      FlatQueues fq, InexactOut out,
                                                      const unsigned long long* __restrict__ row_base) {
  constexpr uint32_t cap = 256u;  // >= kFlatMaxCand
  __shared__ unsigned long long sm[8][cap];
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  unsigned long long* keys = sm[wib];
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const unsigned long long chunk_rows = kSegmentRows ? *row_base : 0ull;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < count; w += nwarps) {
    const uint64_t q = list ? list[q0 + w] : q0 + w;
    const uint32_t sc = fq.seg_cnt[q];
    if (sc == 0xFFFFFFFFu) continue;  // did not fit this pass (already on the retry list)
    const uint32_t cnt = sc & ~kFlatExactBit;
    const uint64_t base = fq.seg_base[q];
    // reserve (or fail) first when the segment is the reservation
    unsigned long long o = chunk_rows + base;
    auto fail = [&]() {  // this pass's buffer is full: retried by the next pass
      if (lane == 0u) {
        const unsigned long long f = atomicAdd(out.fail_count, 1ull);
        out.fail_list[f] = uint32_t(q);
        out.res_cnt[q] = 0u;
      }
    };
    if (kSegmentRows && o + cnt > out.cap) {
      fail();
      continue;
    }
    if (cnt <= 32u) {
      // one candidate per lane: equal intervals found by one match instruction
      uint2 e = make_uint2(1u, 0u);
      if (lane < cnt) e = fq.raw[base + lane];
      const bool alive = e.x <= e.y;
      const unsigned long long key = alive ? ((uint64_t(e.x) << 32) | e.y) : (0xFFFFFFFF00000000ull | lane);
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
      const bool with_exact = (sc & kFlatExactBit) && (peers & 1u);  // lane 0 = W itself
      const bool rep = alive && (with_exact ? lane == 0u : lane == uint32_t(__ffs(peers) - 1));
      const uint32_t repmask = __ballot_sync(0xFFFFFFFFu, rep);
      const uint32_t nuniq = uint32_t(__popc(repmask));
      if (!kSegmentRows) {
        if (lane == 0u && nuniq) o = atomicAdd(out.total, (unsigned long long)nuniq);
        o = __shfl_sync(0xFFFFFFFFu, o, 0);
        if (o + nuniq > out.cap) {
          fail();
          continue;
        }
      }
      uint32_t rank = 0;
      for (uint32_t rest = repmask; rest; rest &= rest - 1u) {
        const unsigned long long kj = __shfl_sync(0xFFFFFFFFu, key, __ffs(rest) - 1);
        rank += kj < key ? 1u : 0u;
      }
      if (rep) {
        out.kl[o + rank] = e;
        out.diffs[o + rank] = with_exact ? uint8_t(0) : uint8_t(1);
      }
      if (lane == 0u) {
        out.res_off[q] = o;
        out.res_cnt[q] = nuniq;
        out.res_pass[q] = out.pass;
      }
      continue;
    }
    // ---- more than 32 candidates survived (patterns inside repeat families):
    // a bitonic sort of the intervals in shared memory, then one pass keeps
    // the first of each (the quadratic rank count this replaces was most of
    // the kernel's instructions on config 3) ----
    // the intervals that exist, compacted (without a filter most of the segment is absent)
    unsigned long long exact_key = ~0ull;  // no interval (k = 0xFFFFFFFF never occurs)
    uint32_t nres = 0;
    __syncwarp();
    for (uint32_t j0 = 0; j0 < cnt; j0 += 32u) {
      uint2 e = make_uint2(1u, 0u);
      if (j0 + lane < cnt) e = fq.raw[base + j0 + lane];
      const bool alive = e.x <= e.y;
      const uint32_t ba = __ballot_sync(0xFFFFFFFFu, alive);
      const unsigned long long x = (uint64_t(e.x) << 32) | e.y;
      if (alive) keys[nres + uint32_t(__popc(ba & lt_mask))] = x;
      if (j0 == 0u && (sc & kFlatExactBit) && (ba & 1u)) exact_key = __shfl_sync(0xFFFFFFFFu, x, 0);  // W itself occurs
      nres += uint32_t(__popc(ba));
    }
    uint32_t P = 32u;
    while (P < nres) P <<= 1;  // nres <= cnt <= kFlatMaxCand < 256
    for (uint32_t j = nres + lane; j < P; j += 32u) keys[j] = ~0ull;  // padding sorts to the end
    __syncwarp();
    for (uint32_t kk = 2u; kk <= P; kk <<= 1) {
      for (uint32_t jj = kk >> 1; jj > 0u; jj >>= 1) {
        for (uint32_t t = lane; t < (P >> 1); t += 32u) {
          const uint32_t i = ((t & ~(jj - 1u)) << 1) | (t & (jj - 1u)), p2 = i | jj;
          const unsigned long long x = keys[i], y = keys[p2];
          if ((x > y) == ((i & kk) == 0u)) {
            keys[i] = y;
            keys[p2] = x;
          }
        }
        __syncwarp();
      }
    }
    // first of each interval, in order: its row is its rank
    uint32_t nuniq = 0;
    if (!kSegmentRows) {
      for (uint32_t j0 = 0; j0 < P; j0 += 32u) {
        const uint32_t j = j0 + lane;
        const unsigned long long x = keys[j];
        const bool first = x != ~0ull && (j == 0u || keys[j - 1u] != x);
        nuniq += uint32_t(__popc(__ballot_sync(0xFFFFFFFFu, first)));
      }
      if (lane == 0u && nuniq) o = atomicAdd(out.total, (unsigned long long)nuniq);
      o = __shfl_sync(0xFFFFFFFFu, o, 0);
      if (o + nuniq > out.cap) {
        fail();
        __syncwarp();
        continue;
      }
      nuniq = 0;
    }
    for (uint32_t j0 = 0; j0 < P; j0 += 32u) {
      const uint32_t j = j0 + lane;
      const unsigned long long x = keys[j];
      const bool first = x != ~0ull && (j == 0u || keys[j - 1u] != x);
      const uint32_t bf = __ballot_sync(0xFFFFFFFFu, first);
      if (first) {
        const uint64_t row = o + nuniq + uint32_t(__popc(bf & lt_mask));
        out.kl[row] = make_uint2(uint32_t(x >> 32), uint32_t(x));
        out.diffs[row] = x == exact_key ? uint8_t(0) : uint8_t(1);
      }
      nuniq += uint32_t(__popc(bf));
    }
    if (lane == 0u) {
      out.res_off[q] = o;
      out.res_cnt[q] = nuniq;
      out.res_pass[q] = out.pass;
    }
    __syncwarp();
  }
}

// Output rows of chunk i start at rows[i]: rows[i + 1] = rows[i] + the queue
// entries chunk i used (its survivor segments double as its rows).  Chunks
// run on several streams; this chain (and the events around it) orders them.
__global__ void k_flat_advance(unsigned long long* rows, const unsigned long long* n_surv, uint64_t q_cap,
                               unsigned long long* total) {
  rows[1] = rows[0] + min(uint64_t(*n_surv), q_cap);
  *total = rows[1];
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
