// Bidirectional z = 1 engine for the bounded-difference search
// (search.py:97-159).  Part of libfmgpu.so (sm_100a); included once by
// fmgpu.cu after kernels_inexact.cuh.
//
// For z = 1 the reference's DFS reports (interval(S), diffs) for every
// string S in the one-edit neighbourhood of W that occurs in the text:
// W itself (diffs 0), one substitution, one deletion (skip), or one
// insertion after W[p] for p in [0, m-1] (never before W[0]); equal
// intervals keep the smallest diffs.  The order of exploration is free, so
// instead of one backward DFS from the empty string — whose wrong-edit
// chains near the right end survive for ~log4(n) characters — the set is
// enumerated in two parts split at h (3m/4 in the split form, m/2 in the
// others; any 0 <= h <= m gives the same set):
//   case A: edits in W[0..h-1] (and insertion after W[h-1]): the right
//     part W[h..m-1] is matched exactly first, then the usual backward DFS
//     runs over the left part on the forward index;
//   case B: edits in W[h..m-1] (insertions after W[p], p >= h): the left
//     part W[0..h-1] is matched exactly first, then a forward DFS runs over
//     the right part on the index of the REVERSED text, with the forward
//     index's interval of S kept in step arithmetically (2BWT):
//     extending S by c on the right, Sc's rows are the rows of S whose next
//     character is c, ordered after "S$" (S a suffix of the text) and after
//     every Sb with b < c, so k(Sc) = k(S) + [S is a text suffix] +
//     sum_{b<c} |Sb| with |Sb| read off the reverse index's Occ step.
// Every chain therefore starts from an already-long exact string and dies
// within a few characters.  Results are the forward-index intervals, so the
// output is bit-identical to the one-directional engines.
#pragma once

#include <cstdint>

#include "occ_device.cuh"

namespace fmg {

struct BiIndex {
  IndexView rev;       // index of the reversed text (same n and C)
  PrefixTable tf, tr;  // prefix tables of the forward / reverse index (same k)
  uint32_t tail[16];   // tail[d]: key of the reversed text's first d characters (d < k), ~0u if d > n
  const uint2* tx = nullptr;  // forward level kx = tf.k + 1 alone (the exact search's k-mer table), or null
  uint32_t kx = 0;
};

// key of W[a .. a+len-1] with W[a] in bits 0..1 (len <= 15)
__device__ __forceinline__ uint32_t pat_key(uint64_t pw0, uint64_t pw1, int a, int len) {
  // branch-free 128-bit funnel shift by 2a: PTX shifts clamp counts >= 64
  // (and the unsigned wrap of a negative count) to an all-zero result
  const uint32_t sh = uint32_t(2 * a);
  uint64_t lo, mid, hi;
  asm("shr.b64 %0, %1, %2;" : "=l"(lo) : "l"(pw0), "r"(sh));
  asm("shl.b64 %0, %1, %2;" : "=l"(mid) : "l"(pw1), "r"(64u - sh));
  asm("shr.b64 %0, %1, %2;" : "=l"(hi) : "l"(pw1), "r"(sh - 64u));
  const uint64_t x = lo | mid | hi;
  return uint32_t(x & ((uint64_t(1) << (2 * len)) - 1u));  // len <= 16
}

__device__ __forceinline__ uint32_t pat_sym(uint64_t pw0, uint64_t pw1, int i) {
  return uint32_t((i < 32 ? pw0 : pw1) >> ((i & 31) << 1)) & 3u;
}

// key of reverse(W[a .. a+len-1]): W[a+len-1] in bits 0..1
__device__ __forceinline__ uint32_t pat_rkey(uint64_t pw0, uint64_t pw1, int a, int len) {
  uint32_t key = 0;
  for (int t = 0; t < len; ++t) key |= pat_sym(pw0, pw1, a + len - 1 - t) << (2 * t);
  return key;
}

// The key of a len-character string read backwards: its 2-bit fields in
// reverse order (len <= 16).
__device__ __forceinline__ uint32_t pair_rev(uint32_t key, uint32_t len) {
  uint32_t v = __brev(key);
  v = ((v >> 1) & 0x55555555u) | ((v & 0x55555555u) << 1);  // bit pairs back in order
  return len == 0u ? 0u : v >> (32u - 2u * len);
}

// The four child intervals of (k, l) on index v: from the prefix table
// (shallow: key, depth) or by one Occ step on the index lines.
template <int W>
__device__ __forceinline__ void children4(const IndexView& v, const PrefixTable& pt, bool shallow, uint32_t x,
                                          uint32_t y, uint32_t ck[4], uint32_t cl[4], uint64_t& work) {
  if (shallow) {
    const uint2* p = pt.base + PrefixTable::off(y + 1u) + 4u * x;
    uint64_t a0, a1, a2, a3;
    ld256<0>(reinterpret_cast<const uint8_t*>(p), a0, a1, a2, a3);
    ck[0] = uint32_t(a0), cl[0] = uint32_t(a0 >> 32), ck[1] = uint32_t(a1), cl[1] = uint32_t(a1 >> 32);
    ck[2] = uint32_t(a2), cl[2] = uint32_t(a2 >> 32), ck[3] = uint32_t(a3), cl[3] = uint32_t(a3 >> 32);
    work += work_unit(1u);
  } else {
    uint32_t lo[4], hi[4];
    work += work_unit(occ_step<W, 0>(v, x, y, lo, hi));
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      ck[b] = v.c[b] + lo[b] + 1u;
      cl[b] = v.c[b] + hi[b];
    }
  }
}

#ifndef FMG_BI_OCC1
#define FMG_BI_OCC1 1  // case-A budget-0 steps count one symbol instead of four
#endif

// kOnly: 0 = both cases per pattern (one result list), 1 = case A only,
// 3 = case B only (phase-uniform launches; k_merge_ab joins the two lists).
#ifndef FMG_BI_JUMP
#define FMG_BI_JUMP 1  // budget-0 chains jump through the prefix tables in one gather
#endif
#ifndef FMG_BI_JUMP_B
// case B too: measured slower (83 -> 104 ms per 14M config-3 seeds) — the
// extra live state makes the case-B kernel spill at 72 registers
#define FMG_BI_JUMP_B 0
#endif
#ifndef FMG_BI_MINB
#define FMG_BI_MINB 7  // resident blocks per SM the register budget is sized for
#endif
#ifndef FMG_BI_NODUP
// Edit paths that spell the same string are expanded once.  Case A (node i,
// string S = edited W[i+1..]): inserting b = W[i] after W[i] gives
// W[0..i] W[i] S, which the match child's insertion of W[i] after W[i-1]
// also gives, so for i >= 1 it is left to node i-1 (at i = 0 there is no
// insertion before W[0]); skipping W[i] when W[i] == W[i-1] gives the string
// that skipping W[i-1] after matching W[i] gives.  Case B mirrors it:
// inserting b = W[j] before W[j] is left to node j+1 (after matching W[j]),
// skipping W[j] when W[j] == W[j+1] is left to node j+1.  The deferred path
// always exists (its lower-bound conditions are weaker, and if its match
// child is empty so is the dropped string), both carry one difference, and
// the result SET is unchanged — the reference's DFS reaches the same strings
// along both paths and keeps one (search.py:128-134).
#define FMG_BI_NODUP 1
#endif

#ifndef FMG_CHAIN_COND_LOW
#define FMG_CHAIN_COND_LOW 1  // k_bchain: load the low line only when it differs from the high one
#endif
#ifndef FMG_BI_PRED_LOW
#define FMG_BI_PRED_LOW 1  // case-A chain steps: predicated low-line load (no request when the line is shared)
#endif
#ifndef FMG_BI_HNUM
// split point h = m * HNUM / 16 of the split DFS form.  Case A (backward:
// one-symbol chain steps, jumps through the tables) is cheaper per edit
// position than case B (forward: four counts per step, no jumps), so the
// split sits right of the middle — config 3 (m = 19), ms per 14M seeds:
// HNUM 8 / 9 / 10 / 11 / 12 / 13 -> 157.6 / 151.3 / 146.6 / 140.9 / 139.4 / 142.5.
#define FMG_BI_HNUM 12
#endif
#ifndef FMG_BI_MINB_A
// the one-word case-A kernel fits 64 registers without spills: 8 blocks per
// SM instead of 7 (config 3 case A 96.3 -> 90.2 ms per 14M seeds)
#define FMG_BI_MINB_A 8
#endif
#ifndef FMG_BI_MINB_B
#define FMG_BI_MINB_B FMG_BI_MINB
#endif

// kOne: every pattern fits one 64-bit word (m <= 32), so the second
// pattern word is the constant 0 (four registers fewer).
template <int W, int kOnly, bool kOne = false>
__global__ void __launch_bounds__(128, kOnly == 3 ? FMG_BI_MINB_B : (kOnly == 1 && kOne) ? FMG_BI_MINB_A : FMG_BI_MINB)
    k_inexact_bi(IndexView ix, BiIndex bi, CodePatterns cp,
                                                    const uint32_t* __restrict__ list, uint64_t count,
                                                    InexactScratch sc, InexactOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t S = sc.S, nt = blockDim.x, tid = threadIdx.x;
  // Stack entries: case A (kOnly == 1) needs only the interval (or key,
  // depth) — 8 bytes + 4 bytes of position/budget; the other forms carry
  // both intervals of case B — 16 + 4 bytes.  Slot S is the push dump.
  constexpr bool kNarrow = kOnly == 1;
  uint4* s_x = reinterpret_cast<uint4*>(smem);                                   // [S + 1][nt] (wide)
  uint2* s_xy = reinterpret_cast<uint2*>(smem);                                  // [S + 1][nt] (narrow)
  uint32_t* s_ib = kNarrow ? reinterpret_cast<uint32_t*>(s_xy + (S + 1) * nt)   // [S + 1][nt]
                           : reinterpret_cast<uint32_t*>(s_x + (S + 1) * nt);
  auto st_put = [&](uint32_t slot, uint32_t x, uint32_t y, uint32_t zz, uint32_t ww) {
    if constexpr (kNarrow) {
      s_xy[slot * nt + tid] = make_uint2(x, y);
    } else {
      s_x[slot * nt + tid] = make_uint4(x, y, zz, ww);
    }
  };
  auto st_get = [&](uint32_t slot) -> uint4 {
    if constexpr (kNarrow) {
      const uint2 v = s_xy[slot * nt + tid];
      return make_uint4(v.x, v.y, 0u, 0u);
    } else {
      return s_x[slot * nt + tid];
    }
  };
  // result sort scratch (the stack is empty by then): (k, l) + diffs
  auto so_put = [&](uint32_t slot, uint32_t k, uint32_t l, uint32_t d) {
    if constexpr (kNarrow) {
      s_xy[slot * nt + tid] = make_uint2(k, l);
      s_ib[slot * nt + tid] = d;
    } else {
      s_x[slot * nt + tid] = make_uint4(k, l, d, 0u);
    }
  };
  auto so_get = [&](uint32_t slot) -> uint4 {
    if constexpr (kNarrow) {
      const uint2 v = s_xy[slot * nt + tid];
      return make_uint4(v.x, v.y, s_ib[slot * nt + tid], 0u);
    } else {
      return s_x[slot * nt + tid];
    }
  };
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= sc.T) return;
  uint64_t my_steps = 0;
  const uint64_t wbase = t >> 5, lane = t & 31u;
  auto HI = [&](uint32_t e) -> uint64_t { return (wbase * (2u * sc.R) + e) * 32u + lane; };
  auto LI = [&](uint32_t e) -> uint64_t { return (wbase * sc.R + e) * 32u + lane; };
  uint32_t epoch = sc.epoch0;
  const uint32_t K = bi.tf.k;
  const uint32_t sent_r = bi.rev.sentinel_row;

  bool have = false;
  uint64_t q = 0;
  int m = 0, h = 0;
  uint64_t pw0 = 0, pw1 = 0, dbits = 0;
  int phase = 1;  // 1: case A (backward, forward index), 3: case B (forward, reverse index)
  uint32_t sp = 0, nres = 0;
  bool overflow = false;
  bool cur_valid = false;
  int ci = 0;                               // i (case A) / j (case B)
  uint32_t cb = 0;                          // budget
  uint32_t cx = 0, cy = 0, cz = 0, cw = 0;  // A: (k, l) or (key, depth); B: F (k, l) + R (k', l') or (rkey, depth)
  bool csh = false;

  auto sym_at = [&](int i) -> uint32_t { return pat_sym(pw0, pw1, i); };
  auto dlb = [&](int i) -> uint32_t { return __popcll(dbits & ((2ull << i) - 1ull)); };
  // (A short contiguous per-thread result list before this table, for case
  // A, saved its probe stalls but the larger kernel lost more to registers:
  // 90.2 -> 97.4 ms per 14M config-3 seeds.)
  auto record = [&](uint32_t k, uint32_t l, uint32_t used) {
    const uint32_t H = 2u * sc.R;
    uint32_t hh = (k * 0x9E3779B1u ^ l * 0x85EBCA77u) & (H - 1u);
    for (uint32_t probe = 0; probe < H; ++probe, hh = (hh + 1u) & (H - 1u)) {
      uint4 e = sc.table[HI(hh)];
      if (e.z != epoch) {
        if (nres == sc.R) {
          overflow = true;
          return;
        }
        sc.table[HI(hh)] = make_uint4(k, l, epoch, used);
        sc.slots[LI(nres)] = hh;
        ++nres;
        return;
      }
      if (e.x == k && e.y == l) {
        if (used < e.w) sc.table[HI(hh)].w = used;
        return;
      }
    }
    overflow = true;
  };
  auto fail = [&]() {
    const unsigned long long f = atomicAdd(out.fail_count, 1ull);
    out.fail_list[f] = uint32_t(q);
    out.res_cnt[q] = kOnly == 0 ? 0u : 0xFFFFFFFFu;  // split launches: k_merge_ab routes it to a retry
  };
  auto finish = [&]() {
    if (overflow) {
      fail();
      return;
    }
    uint64_t o = 0;
    if (nres) {
      o = atomicAdd(out.total, (unsigned long long)nres);
      if (o + nres > out.cap) {
        fail();
        return;
      }
      if (nres <= S) {  // insertion sort by (k, l) in the (empty) stack slots
        for (uint32_t r = 0; r < nres; ++r) {
          const uint4 e = sc.table[HI(sc.slots[LI(r)])];
          uint32_t b = r;
          while (b > 0) {
            const uint4 p = so_get(b - 1);
            if (p.x < e.x || (p.x == e.x && p.y < e.y)) break;
            so_put(b, p.x, p.y, p.z);
            --b;
          }
          so_put(b, e.x, e.y, e.w);
        }
        for (uint32_t r = 0; r < nres; ++r) {
          const uint4 p = so_get(r);
          out.kl[o + r] = make_uint2(p.x, p.y);
          out.diffs[o + r] = uint8_t(p.z);
        }
      } else {
        for (uint32_t r = 0; r < nres; ++r) {
          const uint4 e = sc.table[HI(sc.slots[LI(r)])];
          out.kl[o + r] = make_uint2(e.x, e.y);
          out.diffs[o + r] = uint8_t(e.w);
        }
        const unsigned long long u = atomicAdd(out.unsorted, 1ull);
        out.unsorted_list[u] = uint32_t(q);
      }
    }
    out.res_off[q] = o;
    out.res_cnt[q] = nres;
    out.res_pass[q] = out.pass;
  };
  auto push_if = [&](bool cond, int pos, uint32_t pb, bool psh, uint32_t x, uint32_t y, uint32_t zz, uint32_t ww) {
    const bool ok = cond && sp < S;
    overflow |= cond && sp >= S;
    const uint32_t slot = ok ? sp : S;
    st_put(slot, x, y, zz, ww);
    s_ib[slot * nt + tid] = (uint32_t(pos + 1) << 16) | (psh ? 0x8000u : 0u) | pb;
    sp += ok ? 1u : 0u;
  };

  // case A root: interval of W[h..m-1], then node (h-1, budget 1)
  auto root_a = [&]() -> bool {
    const int r = m - h;
    const int tt = min(r, int(K));
    uint2 e = __ldg(bi.tf.base + PrefixTable::off(uint32_t(tt)) + pat_key(pw0, pw1, m - tt, tt));
    my_steps += work_unit(1u);
    for (int p = m - tt - 1; p >= h && e.x <= e.y; --p) {
      uint32_t ck[4], cl[4];
      children4<W>(ix, bi.tf, false, e.x, e.y, ck, cl, my_steps);
      const uint32_t b = sym_at(p);
      e = make_uint2(sel4(ck, b), sel4(cl, b));
    }
    if (e.x > e.y) return false;
    if (h == 0) {  // the whole pattern matched: the exact result
      record(e.x, e.y, 0u);
      return false;
    }
    if (dlb(h - 1) > 1u) return false;
    ci = h - 1;
    cb = 1u;
    csh = uint32_t(r) < K;
    cx = csh ? pat_key(pw0, pw1, h, r) : e.x;
    cy = csh ? uint32_t(r) : e.y;
    return true;
  };
  // case B root: both intervals of W[0..h-1], then node (h, budget 1)
  auto root_b = [&]() -> bool {
    const int tt = min(h, int(K));
    uint2 f = make_uint2(0u, ix.n), rr = make_uint2(0u, ix.n);
    if (tt > 0) {
      f = __ldg(bi.tf.base + PrefixTable::off(uint32_t(tt)) + pat_key(pw0, pw1, 0, tt));
      rr = __ldg(bi.tr.base + PrefixTable::off(uint32_t(tt)) + pat_rkey(pw0, pw1, 0, tt));
      my_steps += work_unit(2u);
    }
    for (int p = tt; p < h && f.x <= f.y; ++p) {
      uint32_t rk[4], rl[4];
      children4<W>(bi.rev, bi.tr, false, rr.x, rr.y, rk, rl, my_steps);
      const uint32_t w = sym_at(p);
      uint32_t k = f.x + ((rr.x <= sent_r && sent_r <= rr.y) ? 1u : 0u);
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (b < w) k += rl[b] + 1u - rk[b];
      const uint32_t sz = sel4(rl, w) + 1u - sel4(rk, w);
      f = make_uint2(k, k + sz - 1u);
      rr = make_uint2(sel4(rk, w), sel4(rl, w));
      if (sz == 0u) f = make_uint2(1u, 0u);
    }
    if (f.x > f.y) return false;
    ci = h;
    cb = 1u;
    csh = uint32_t(h) < K;
    cx = f.x;
    cy = f.y;
    cz = csh ? pat_rkey(pw0, pw1, 0, h) : rr.x;
    cw = csh ? uint32_t(h) : rr.y;
    return true;
  };

  // The next pattern is claimed and its words loaded while the current one
  // is searched, so starting a pattern never waits on the queue atomic and
  // the pattern loads (they would stall the whole warp for the lanes that
  // start).
  uint64_t nq = 0, npw0 = 0, npw1 = 0, ndbits = 0;
  int nm = 0;
  bool nvalid = false;
  auto prefetch = [&]() {
    const unsigned long long slot = atomicAdd(out.next, 1ull);
    nvalid = slot < count;
    if (!nvalid) return;
    nq = list ? list[slot] : slot;
    if (cp.packed1) {
      nm = int(cp.fixed_m);
      npw0 = cp.packed1[nq];
      npw1 = 0;
    } else if (kOne) {
      nm = int(cp.offsets[nq + 1] - cp.offsets[nq]);
      npw0 = cp.packed[nq].x;
      npw1 = 0;
    } else {
      nm = int(cp.offsets[nq + 1] - cp.offsets[nq]);
      const ulonglong2 pk = cp.packed[nq];
      npw0 = pk.x;
      npw1 = pk.y;
    }
    ndbits = cp.dbits[nq];
  };
  prefetch();

  while (true) {
    bool stepping = false;
    while (!stepping) {
      if (!have) {
        if (!nvalid) break;
        q = nq;
        m = nm;
        pw0 = npw0;
        pw1 = kOne ? 0ull : npw1;
        dbits = ndbits;
        prefetch();
        h = (m * FMG_BI_HNUM) / 16;  // split point: case A edits W[0..h-1], case B W[h..m-1]
        sp = nres = 0;
        ++epoch;
        overflow = false;
        phase = kOnly == 3 ? 3 : 1;
        have = true;
        cur_valid = dlb(m - 1) <= 1u && (kOnly == 3 ? root_b() : root_a());
      }
      if (overflow) {
        finish();
        have = false;
        continue;
      }
      if (!cur_valid) {
        if (sp > 0) {
          --sp;
          const uint4 e = st_get(sp);
          const uint32_t ib = s_ib[sp * nt + tid];
          ci = int(ib >> 16) - 1;
          cb = ib & 0xFFu;
          csh = (ib >> 15) & 1u;
          cx = e.x;
          cy = e.y;
          cz = e.z;
          cw = e.w;
          cur_valid = true;
          // (An L2 prefetch of the new stack top's first access at each pop
          // measured slower: case A 90.2 -> 98.2 ms per 14M config-3 seeds.)
        } else if (kOnly == 0 && phase == 1) {
          phase = 3;
          cur_valid = dlb(m - 1) <= 1u && root_b();
          continue;
        } else {
          finish();
          have = false;
          continue;
        }
      }
      stepping = true;
    }
    if (!stepping) break;

    // ---- budget-0 node inside the prefix tables' depth range: jump ----
    // Its string grows by known pattern characters only, so the node t =
    // min(characters left, K - depth) levels down is ONE table gather away
    // instead of t dependent ones.  Case A prepends W[i], W[i-1], ... (key
    // of W[i-t+1..i] below the node's key); case B appends W[j..j+t-1]: the
    // reverse key grows the same way and the forward interval is read from
    // the forward table under the bit-pair-reversed key (for a non-empty
    // string the table entry IS the interval the 2BWT update computes; an
    // empty one ends the chain either way).  Chains that reach depth K
    // continue on the index lines with explicit intervals.
    constexpr bool kJumpA = FMG_BI_JUMP && kOnly != 3, kJumpB = FMG_BI_JUMP_B && kOnly != 1;
    if (cb == 0u && csh && ((kJumpA && phase != 3) || (kJumpB && phase == 3))) {
      if (phase != 3) {  // case A; with the level-(K+1) table the jump lands one level deeper
        const uint32_t kmax = bi.tx ? bi.kx : K;
        const uint32_t t = min(uint32_t(ci) + 1u, kmax - cy);
        const uint32_t d = cy + t;
        const uint32_t key = pat_key(pw0, pw1, ci - int(t) + 1, int(t)) | uint32_t(uint64_t(cx) << (2u * t));
        const uint2 e = __ldg(d > K ? bi.tx + key : bi.tf.base + PrefixTable::off(d) + key);
        // (Also gathering the final string's first K + 1 characters beside
        // `e`, to end absent chains here, measured slower: 96.3 -> 99.9 ms.)
        my_steps += work_unit(1u);
        if (e.x > e.y) {
          cur_valid = false;
        } else if (uint32_t(ci) + 1u == t) {
          record(e.x, e.y, 1u);
          cur_valid = false;
        } else {
          ci -= int(t);
          cx = e.x;
          cy = e.y;
          csh = false;
          cur_valid = dlb(ci) == 0u;
        }
      } else {  // case B
        const uint32_t t = min(uint32_t(m - ci), K - cw);
        const uint32_t d = cw + t;
        // forward key of S = the node's reverse key with its bit pairs
        // reversed; S' = S + W[j..j+t-1] appends the pattern's key above it
        const uint32_t fkey = pair_rev(cz, cw) | (pat_key(pw0, pw1, ci, int(t)) << (2u * cw));
        const uint2 f = __ldg(bi.tf.base + PrefixTable::off(d) + fkey);
        const bool done = uint32_t(m - ci) == t;
        uint2 r = make_uint2(0u, 0u);
        if (!done) r = __ldg(bi.tr.base + PrefixTable::off(d) + pair_rev(fkey, d));
        my_steps += work_unit(done ? 1u : 2u);
        if (f.x > f.y) {
          cur_valid = false;
        } else if (done) {
          record(f.x, f.y, 1u);
          cur_valid = false;
        } else {
          ci += int(t);
          cx = f.x;
          cy = f.y;
          cz = r.x;
          cw = r.y;
          csh = false;
        }
      }
      continue;
    }

    // ---- one step: the four children of the node's string ----
    // (a compile-time `fwd` for the split launches measured slower: case B
    // 83 -> 99 ms per 14M config-3 seeds, register spills)
    const bool fwd = phase == 3;
    uint32_t ck[4], cl[4];
    // (One shared pair of loads for every node kind, selecting addresses
    // first, measured no faster for case A and slower for case B: 79.6 ->
    // 79.1 ms and 83.5 -> 97 ms per 14M config-3 seeds.)
    // (A case-B budget-0 step from Occ of W[j] plus the count of the symbols
    // below it, instead of all four counts, measured slower: 83 -> 137 ms
    // per 14M config-3 seeds, spills at 72 registers.)
#if FMG_BI_OCC1
    // case-A budget-0 node: only the symbol W[i] is needed (one-symbol count)
    const bool one = !fwd && cb == 0u && !csh;
    uint32_t k1 = 0, l1 = 0;
    if (one) {
      const uint32_t sym = sym_at(ci);
      constexpr uint32_t kC = LineTraits<W>::kChars;
      const uint32_t low = cx - 1u;
      const uint32_t jh = line_of<W>(cy), jl = line_of<W>(low);
      uint32_t bh[4], bl[4];
      uint64_t wh[W], wl[W];
      load_line<W, 0>(ix, jh, cy - jh * kC, bh, wh);
      if constexpr (W == 2 && FMG_BI_PRED_LOW && kOnly == 1) {
        // the low line is loaded only when it differs (deep chains: nearly
        // always the same line, and a second load is a second request)
        uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        ld256_pred(jl != jh, ix.lines + size_t(jl) * LineTraits<2>::kBytes, a0, a1, a2, a3);
        const bool same = jl == jh;
        bl[0] = same ? bh[0] : uint32_t(a0);
        bl[1] = same ? bh[1] : uint32_t(a0 >> 32);
        bl[2] = same ? bh[2] : uint32_t(a1);
        bl[3] = same ? bh[3] : uint32_t(a1 >> 32);
        wl[0] = same ? wh[0] : a2;
        wl[1] = same ? wh[1] : a3;
      } else {
        load_line<W, 0>(ix, jl, low - jl * kC, bl, wl);
      }
      const uint32_t cs = c_of(ix, sym);
      k1 = cs + occ1_from_line<W>(ix, bl, wl, low, low - jl * kC, sym) + 1u;
      l1 = cs + occ1_from_line<W>(ix, bh, wh, cy, cy - jh * kC, sym);
      my_steps += work_unit(jl != jh ? 2u : 1u);
    } else {
      children4<W>(fwd ? bi.rev : ix, fwd ? bi.tr : bi.tf, csh, fwd ? cz : cx, fwd ? cw : cy, ck, cl, my_steps);
    }
#else
    constexpr bool one = false;
    uint32_t k1 = 0, l1 = 0;
    children4<W>(fwd ? bi.rev : ix, fwd ? bi.tr : bi.tf, csh, fwd ? cz : cx, fwd ? cw : cy, ck, cl, my_steps);
#endif

    if (!fwd) {
      // ---- case A: backward expansion (search.py:135-152) ----
      const int i = ci;
      const uint32_t want = sym_at(i);
      const uint32_t kw = one ? k1 : sel4(ck, want), lw = one ? l1 : sel4(cl, want);
      const bool child_sh = csh && cy + 1u < K;
      if (cb == 0u) {
        if (kw > lw) {
          cur_valid = false;
        } else if (i == 0) {
          record(kw, lw, 1u);
          cur_valid = false;
        } else {
          ci = i - 1;
          cx = child_sh ? want + 4u * cx : kw;
          cy = child_sh ? cy + 1u : lw;
          csh = child_sh;
          cur_valid = dlb(i - 1) == 0u;
        }
        continue;
      }
      const bool at0 = i == 0;
      const uint32_t d_prev = at0 ? 0u : dlb(i - 1), d_cur = dlb(i);
      const bool ok_match = !at0 && d_prev <= 1u;
      const bool ok_prev = !at0 && d_prev == 0u;
      const bool ok_cur = d_cur == 0u;
      if (at0) {
        if (kw <= lw) record(kw, lw, 0u);
        uint32_t sk = cx, sl = cy;  // skip: this node's own interval
        if (csh) {
          if (cy == 0u) {
            sk = 0u;
            sl = ix.n;
          } else {
            const uint2 e = __ldg(bi.tf.base + PrefixTable::off(cy) + cx);
            sk = e.x;
            sl = e.y;
          }
        }
        record(sk, sl, 1u);
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b)
          if (b != want && ck[b] <= cl[b]) record(ck[b], cl[b], 1u);  // mismatch
      }
      const uint32_t ckey = 4u * cx, cdep = cy + 1u;
      push_if(ok_match && kw <= lw, i - 1, 1u, child_sh, child_sh ? want + ckey : kw, child_sh ? cdep : lw, 0u, 0u);
      const bool skip_ok = ok_prev && (!FMG_BI_NODUP || want != sym_at(i - 1));
      push_if(skip_ok, i - 1, 0u, csh, cx, cy, 0u, 0u);  // skip
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b) {
        const bool ne = ck[b] <= cl[b];
        const uint32_t px = child_sh ? b + ckey : ck[b], py = child_sh ? cdep : cl[b];
        const bool ins_ok = !FMG_BI_NODUP || b != want || at0;
        push_if(ok_cur && ne && ins_ok, i, 0u, child_sh, px, py, 0u, 0u);        // insert
        push_if(ok_prev && ne && b != want, i - 1, 0u, child_sh, px, py, 0u, 0u);  // mismatch
      }
      cur_valid = false;
      continue;
    }

    // ---- case B: forward expansion on the reverse index ----
    const int j = ci;
    uint32_t sz[4], fk[4];
    const bool dollar = csh ? (cz == bi.tail[cw]) : (cz <= sent_r && sent_r <= cw);
    uint32_t acc = cx + (dollar ? 1u : 0u);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      sz[b] = cl[b] + 1u - ck[b];
      fk[b] = acc;
      acc += sz[b];
    }
    const bool child_sh = csh && cw + 1u < K;
    const uint32_t rkey = 4u * cz, rdep = cw + 1u;
    auto cz_of = [&](uint32_t b) { return child_sh ? b + rkey : sel4(ck, b); };
    auto cw_of = [&](uint32_t b) { return child_sh ? rdep : sel4(cl, b); };
    if (cb == 0u) {  // only the match child; j < m here
      const uint32_t w = sym_at(j);
      const uint32_t s = sel4(sz, w), k = sel4(fk, w);
      if (s == 0u) {
        cur_valid = false;
      } else if (j + 1 == m) {
        record(k, k + s - 1u, 1u);
        cur_valid = false;
      } else {
        ci = j + 1;
        cz = cz_of(w);
        cw = cw_of(w);
        cx = k;
        cy = k + s - 1u;
        csh = child_sh;
      }
      continue;
    }
    if (j == m) {  // budget 1 after the whole pattern: insertion after W[m-1]
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (sz[b]) record(fk[b], fk[b] + sz[b] - 1u, 1u);
      cur_valid = false;
      continue;
    }
    const uint32_t w = sym_at(j);
    const bool last = j + 1 == m;
    const uint32_t sw = sel4(sz, w), kw = sel4(fk, w);
    if (last) {
      if (sw) record(kw, kw + sw - 1u, 0u);  // W itself (also found by case A)
      record(cx, cy, 1u);                    // skip W[m-1]
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (b != w && sz[b]) record(fk[b], fk[b] + sz[b] - 1u, 1u);  // mismatch at m-1
    }
    // match: (j+1, 1); at the end it still expands for insertions after W[m-1]
    push_if(sw != 0u, j + 1, 1u, child_sh, kw, kw + sw - 1u, cz_of(w), cw_of(w));
    push_if(!last && (!FMG_BI_NODUP || w != sym_at(j + 1)), j + 1, 0u, csh, cx, cy, cz, cw);  // skip
    const bool ins = j >= h + 1;                      // insertion after W[j-1], j-1 >= h
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b) {
      const bool ne = sz[b] != 0u;
      const uint32_t px = child_sh ? b + rkey : ck[b], py = child_sh ? rdep : cl[b];
      push_if(!last && ne && b != w, j + 1, 0u, child_sh, fk[b], fk[b] + sz[b] - 1u, px, py);  // mismatch
      push_if(ins && ne && (!FMG_BI_NODUP || b != w), j, 0u, child_sh, fk[b], fk[b] + sz[b] - 1u, px,
              py);  // insert
    }
    cur_valid = false;
  }
  flush_work(out.steps, my_steps);
}

// Joins the case-A and case-B result lists of each pattern (each sorted by
// (k, l), unique within itself): merge, equal intervals keep the smaller
// diffs.  Count pass (write == false) then write pass into one buffer.
// A pattern whose A or B launch failed (res_cnt ~0) gets count 0 here and
// is appended to `retry` for the one-directional DFS engine.
__global__ void k_merge_ab(uint64_t count, const uint64_t* __restrict__ offA, const uint32_t* __restrict__ cntA,
                           const uint2* __restrict__ klA, const uint8_t* __restrict__ dA,
                           const uint64_t* __restrict__ offB, const uint32_t* __restrict__ cntB,
                           const uint2* __restrict__ klB, const uint8_t* __restrict__ dB, bool write,
                           uint64_t* __restrict__ c64, const uint64_t* __restrict__ out_off, uint2* __restrict__ kl,
                           uint8_t* __restrict__ dd, uint32_t* __restrict__ res_cnt, uint64_t* __restrict__ res_off,
                           uint8_t* __restrict__ res_pass, uint32_t* __restrict__ retry,
                           unsigned long long* __restrict__ n_retry) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint32_t na = cntA[q], nb = cntB[q];
  if (na == 0xFFFFFFFFu || nb == 0xFFFFFFFFu) {
    if (write) {
      res_cnt[q] = 0;
      const unsigned long long r = atomicAdd(n_retry, 1ull);
      retry[r] = uint32_t(q);
    } else {
      c64[q] = 0;
    }
    return;
  }
  const uint2* a = klA + (na ? offA[q] : 0);
  const uint2* b = klB + (nb ? offB[q] : 0);
  const uint8_t* da = dA + (na ? offA[q] : 0);
  const uint8_t* db = dB + (nb ? offB[q] : 0);
  uint64_t o = write ? out_off[q] : 0;
  uint32_t i = 0, j = 0, n = 0;
  while (i < na || j < nb) {
    uint2 x;
    uint8_t d;
    if (j >= nb || (i < na && (a[i].x < b[j].x || (a[i].x == b[j].x && a[i].y < b[j].y)))) {
      x = a[i];
      d = da[i++];
    } else if (i >= na || (a[i].x != b[j].x || a[i].y != b[j].y)) {
      x = b[j];
      d = db[j++];
    } else {  // the same interval from both halves
      x = a[i];
      d = min(da[i], db[j]);
      ++i;
      ++j;
    }
    if (write) {
      kl[o + n] = x;
      dd[o + n] = d;
    }
    ++n;
  }
  if (write) {
    res_cnt[q] = n;
    res_off[q] = o;
    res_pass[q] = 0;
  } else {
    c64[q] = n;
  }
}

// ----- level-synchronous form (the default bidirectional engine) ----------
//
// k_bspine: one thread per pattern walks both budget-1 spines — case A over
// W[h-1..0] on the forward index, case B over W[h..m-1] on the reverse
// index — queuing every budget-0 child as a Z1BNode and writing results
// reached at the pattern ends as Z1Raw.  Patterns of equal length keep the
// warp in lock-step.  k_bchain: persistent lane-refill over the queued
// nodes, each an exact extension (backward for case A, forward for case B)
// until its string leaves the text or the pattern ends.  Deduplication and
// ordering reuse the z1 engine's kernels.
struct Z1BNode {  // a budget-0 continuation of pattern q
  uint32_t q;
  uint32_t pos;  // bits 0..15: next position; bit 16: case B (forward); bit 17: shallow
  uint32_t x, y, zz, ww;  // A: (k, l) | (key, depth); B: F (k, l) + R (k', l') | (rkey, depth)
};
struct Z1BQueues {
  Z1BNode* nodes;
  unsigned long long* n_nodes;
  uint64_t node_cap;
  Z1Raw* raws;
  unsigned long long* n_raws;
  uint64_t raw_cap;
};

__device__ __forceinline__ void z1b_pattern(const CodePatterns& cp, uint64_t q, uint64_t& pw0, uint64_t& pw1,
                                            int& m) {
  if (cp.packed1) {
    pw0 = cp.packed1[q];
    pw1 = 0;
    m = int(cp.fixed_m);
  } else {
    const ulonglong2 pk = cp.packed[q];
    pw0 = pk.x;
    pw1 = pk.y;
    m = int(cp.offsets[q + 1] - cp.offsets[q]);
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_bspine(IndexView ix, BiIndex bi, CodePatterns cp, uint64_t q0,
                                                uint64_t count, Z1BQueues qu, unsigned long long* steps) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const uint32_t q = uint32_t(q0 + t);
  uint64_t pw0, pw1;
  int m;
  z1b_pattern(cp, q, pw0, pw1, m);
  const uint64_t dbits = cp.dbits[q];
  auto dlb = [&](int i) -> uint32_t { return __popcll(dbits & ((2ull << i) - 1ull)); };
  uint64_t work = 0;
  const uint32_t K = bi.tf.k;
  const uint32_t sent_r = bi.rev.sentinel_row;
  const int h = m / 2;
  auto raw = [&](bool c, uint32_t k, uint32_t l, uint32_t used, uint64_t& slot) {
    if (c) {
      if (slot < qu.raw_cap) qu.raws[slot] = Z1Raw{q, k, l, used};
      ++slot;
    }
  };
  auto node = [&](bool c, uint32_t pos, uint32_t x, uint32_t y, uint32_t zz, uint32_t ww, uint64_t& slot) {
    if (c) {
      if (slot < qu.node_cap) qu.nodes[slot] = Z1BNode{q, pos, x, y, zz, ww};
      ++slot;
    }
  };
  if (dlb(m - 1) > 1u) {  // two absent segments: no string within one edit occurs
    flush_work(steps, work);
    return;
  }

  // ---- case A: W[h..m-1] exactly, then the backward spine over W[h-1..0] ----
  {
    const int r = m - h;
    const int tt = min(r, int(K));
    uint2 e = __ldg(bi.tf.base + PrefixTable::off(uint32_t(tt)) + pat_key(pw0, pw1, m - tt, tt));
    work += work_unit(1u);
    for (int p = m - tt - 1; p >= h && e.x <= e.y; --p) {
      uint32_t ck[4], cl[4];
      children4<W>(ix, bi.tf, false, e.x, e.y, ck, cl, work);
      const uint32_t b = pat_sym(pw0, pw1, p);
      e = make_uint2(sel4(ck, b), sel4(cl, b));
    }
    bool alive = e.x <= e.y;
    if (alive && h == 0) {
      uint64_t rs = warp_reserve(qu.n_raws, 1u);
      raw(true, e.x, e.y, 0u, rs);
      alive = false;
    }
    alive = alive && dlb(h - 1) <= 1u;
    bool sh = uint32_t(r) < K;
    uint32_t x = sh ? pat_key(pw0, pw1, h, r) : e.x, y = sh ? uint32_t(r) : e.y;
    int i = h - 1;
    while (alive) {
      uint32_t ck[4], cl[4];
      children4<W>(ix, bi.tf, sh, x, y, ck, cl, work);
      const uint32_t want = pat_sym(pw0, pw1, i);
      const bool at0 = i == 0;
      const bool ok_prev = !at0 && dlb(i - 1) == 0u, ok_cur = dlb(i) == 0u;
      const bool child_sh = sh && y + 1u < K;
      uint32_t e_ins = 0, e_mis = 0;
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b) {
        const bool ne = ck[b] <= cl[b];
        e_ins |= (ok_cur && ne && (!FMG_BI_NODUP || b != want || at0)) ? (1u << b) : 0u;
        e_mis |= (ok_prev && ne && b != want) ? (1u << b) : 0u;
      }
      const bool skip_ok = ok_prev && (!FMG_BI_NODUP || want != pat_sym(pw0, pw1, i - 1));
      uint64_t slot = warp_reserve(qu.n_nodes, (skip_ok ? 1u : 0u) + __popc(e_ins) + __popc(e_mis));
      node(skip_ok, uint32_t(i - 1) | (sh ? 0x20000u : 0u), x, y, 0u, 0u, slot);  // skip
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b) {
        const uint32_t px = child_sh ? b + 4u * x : ck[b], py = child_sh ? y + 1u : cl[b];
        const uint32_t fl = child_sh ? 0x20000u : 0u;
        node((e_ins >> b) & 1u, uint32_t(i) | fl, px, py, 0u, 0u, slot);      // insert
        node((e_mis >> b) & 1u, uint32_t(i - 1) | fl, px, py, 0u, 0u, slot);  // mismatch
      }
      const uint32_t kw = sel4(ck, want), lw = sel4(cl, want);
      // results at the left end (search.py:127-134): rare
      uint32_t n_at0 = 0;
      if (at0) {
        n_at0 = (kw <= lw ? 1u : 0u) + 1u;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) n_at0 += (b != want && ck[b] <= cl[b]) ? 1u : 0u;
      }
      uint64_t rs = warp_reserve(qu.n_raws, n_at0);
      if (at0) {
        raw(kw <= lw, kw, lw, 0u, rs);
        uint32_t sk = x, sl = y;  // skip: this node's own interval
        if (sh) {
          if (y == 0u) {
            sk = 0u;
            sl = ix.n;
          } else {
            const uint2 o = __ldg(bi.tf.base + PrefixTable::off(y) + x);
            sk = o.x;
            sl = o.y;
          }
        }
        raw(true, sk, sl, 1u, rs);
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) raw(b != want && ck[b] <= cl[b], ck[b], cl[b], 1u, rs);
        break;
      }
      if (kw > lw || dlb(i - 1) > 1u) break;
      x = child_sh ? want + 4u * x : kw;
      y = child_sh ? y + 1u : lw;
      sh = child_sh;
      --i;
    }
  }

  // ---- case B: W[0..h-1] exactly, then the forward spine over W[h..m-1] ----
  {
    const int tt = min(h, int(K));
    uint2 f = make_uint2(0u, ix.n), rr = make_uint2(0u, ix.n);
    if (tt > 0) {
      f = __ldg(bi.tf.base + PrefixTable::off(uint32_t(tt)) + pat_key(pw0, pw1, 0, tt));
      rr = __ldg(bi.tr.base + PrefixTable::off(uint32_t(tt)) + pat_rkey(pw0, pw1, 0, tt));
      work += work_unit(2u);
    }
    for (int p = tt; p < h && f.x <= f.y; ++p) {
      uint32_t rk[4], rl[4];
      children4<W>(bi.rev, bi.tr, false, rr.x, rr.y, rk, rl, work);
      const uint32_t w = pat_sym(pw0, pw1, p);
      uint32_t k = f.x + ((rr.x <= sent_r && sent_r <= rr.y) ? 1u : 0u);
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (b < w) k += rl[b] + 1u - rk[b];
      const uint32_t sz = sel4(rl, w) + 1u - sel4(rk, w);
      f = sz ? make_uint2(k, k + sz - 1u) : make_uint2(1u, 0u);
      rr = make_uint2(sel4(rk, w), sel4(rl, w));
    }
    bool alive = f.x <= f.y;
    bool sh = uint32_t(h) < K;
    uint32_t fx = f.x, fy = f.y;
    uint32_t rz = sh ? pat_rkey(pw0, pw1, 0, h) : rr.x, rw = sh ? uint32_t(h) : rr.y;
    int j = h;
    while (alive) {
      uint32_t ck[4], cl[4];
      children4<W>(bi.rev, bi.tr, sh, rz, rw, ck, cl, work);
      const bool dollar = sh ? (rz == bi.tail[rw]) : (rz <= sent_r && sent_r <= rw);
      uint32_t sz[4], fk[4];
      uint32_t acc = fx + (dollar ? 1u : 0u);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        sz[b] = cl[b] + 1u - ck[b];
        fk[b] = acc;
        acc += sz[b];
      }
      const bool child_sh = sh && rw + 1u < K;
      const uint32_t fl = 0x10000u | (child_sh ? 0x20000u : 0u);
      if (j == m) {  // insertion after W[m-1]
        uint32_t n_ins = 0;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) n_ins += sz[b] ? 1u : 0u;
        uint64_t rs = warp_reserve(qu.n_raws, n_ins);
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) raw(sz[b] != 0u, fk[b], fk[b] + sz[b] - 1u, 1u, rs);
        break;
      }
      const uint32_t w = pat_sym(pw0, pw1, j);
      const bool last = j + 1 == m;
      const bool ins = j >= h + 1;  // insertion after W[j-1], j-1 >= h
      uint32_t e_ins = 0, e_mis = 0;
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b) {
        e_ins |= (ins && sz[b] && (!FMG_BI_NODUP || b != w)) ? (1u << b) : 0u;
        e_mis |= (!last && sz[b] && b != w) ? (1u << b) : 0u;
      }
      const bool skip_ok = !last && (!FMG_BI_NODUP || w != pat_sym(pw0, pw1, j + 1));
      uint64_t slot = warp_reserve(qu.n_nodes, (skip_ok ? 1u : 0u) + __popc(e_ins) + __popc(e_mis));
      node(skip_ok, uint32_t(j + 1) | 0x10000u | (sh ? 0x20000u : 0u), fx, fy, rz, rw, slot);  // skip
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b) {
        const uint32_t pz = child_sh ? b + 4u * rz : ck[b], pw = child_sh ? rw + 1u : cl[b];
        node((e_mis >> b) & 1u, uint32_t(j + 1) | fl, fk[b], fk[b] + sz[b] - 1u, pz, pw, slot);  // mismatch
        node((e_ins >> b) & 1u, uint32_t(j) | fl, fk[b], fk[b] + sz[b] - 1u, pz, pw, slot);      // insert
      }
      const uint32_t sw = sel4(sz, w), kw = sel4(fk, w);
      uint32_t n_last = 0;
      if (last) {
        n_last = (sw ? 1u : 0u) + 1u;
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) n_last += (b != w && sz[b]) ? 1u : 0u;
      }
      uint64_t rs = warp_reserve(qu.n_raws, n_last);
      if (last) {
        raw(sw != 0u, kw, kw + sw - 1u, 0u, rs);  // W itself (also found by case A)
        raw(true, fx, fy, 1u, rs);                // skip W[m-1]
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) raw(b != w && sz[b], fk[b], fk[b] + sz[b] - 1u, 1u, rs);  // mismatch
      }
      if (sw == 0u) break;
      // the match child; after W[m-1] it still expands once for the insertions
      rz = child_sh ? w + 4u * rz : sel4(ck, w);
      rw = child_sh ? rw + 1u : sel4(cl, w);
      fx = kw;
      fy = kw + sw - 1u;
      sh = child_sh;
      ++j;
    }
  }
  flush_work(steps, work);
}

template <int W>
__global__ void __launch_bounds__(256) k_bchain(IndexView ix, BiIndex bi, CodePatterns cp,
                                                const Z1BNode* __restrict__ nodes,
                                                const unsigned long long* __restrict__ n_nodes_dev, Z1BQueues qu,
                                                unsigned long long* steps) {
  // the queue length k_bspine left on the device (no host round trip)
  const uint64_t n_nodes = min(uint64_t(*n_nodes_dev), qu.node_cap);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t work = 0;
  const uint32_t K = bi.tf.k;
  const uint32_t sent_r = bi.rev.sentinel_row;
  uint64_t pw0 = 0, pw1 = 0, dbits = 0;
  int m = 0, pos = 0;
  uint32_t q = 0, x = 0, y = 0, zz = 0, ww = 0;
  bool fwd = false, sh = false, have = false;
  while (true) {
    if (!have) {
      if (t >= n_nodes) break;
      const Z1BNode nd = nodes[t];
      t += stride;
      q = nd.q;
      z1b_pattern(cp, q, pw0, pw1, m);
      dbits = cp.dbits[q];
      pos = int(nd.pos & 0xFFFFu);
      fwd = (nd.pos >> 16) & 1u;
      sh = (nd.pos >> 17) & 1u;
      x = nd.x;
      y = nd.y;
      zz = nd.zz;
      ww = nd.ww;
      have = true;
    }
    // A chain inside the prefix tables' depth range grows by known pattern
    // characters only: jump to the deepest table level it reaches in one
    // gather (case A: into the level-(K+1) table when built; case B: the
    // forward interval from the forward table under the bit-pair-reversed
    // key, the reverse interval only if the chain goes on).
    if (sh && FMG_BI_JUMP) {
      if (!fwd) {
        const uint32_t kmax = bi.tx ? bi.kx : K;
        const uint32_t tt = min(uint32_t(pos) + 1u, kmax - y);
        const uint32_t d = y + tt;
        const uint32_t key = pat_key(pw0, pw1, pos - int(tt) + 1, int(tt)) | uint32_t(uint64_t(x) << (2u * tt));
        const uint2 e = __ldg(d > K ? bi.tx + key : bi.tf.base + PrefixTable::off(d) + key);
        work += work_unit(1u);
        const bool done = uint32_t(pos) + 1u == tt;
        if (e.x > e.y || done) {
          have = false;
          if (e.x <= e.y) {
            const unsigned long long rs = atomicAdd(qu.n_raws, 1ull);
            if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{q, e.x, e.y, 1u};
          }
          continue;
        }
        pos -= int(tt);
        if (__popcll(dbits & ((2ull << pos) - 1ull)) > 0u) {  // an absent segment in W[0..pos]
          have = false;
          continue;
        }
        x = e.x;
        y = e.y;
        sh = false;
      } else {
        const uint32_t tt = min(uint32_t(m - pos), K - ww);
        const uint32_t d = ww + tt;
        const uint32_t fkey = pair_rev(zz, ww) | (pat_key(pw0, pw1, pos, int(tt)) << (2u * ww));
        const uint2 f = __ldg(bi.tf.base + PrefixTable::off(d) + fkey);
        const bool done = uint32_t(m - pos) == tt;
        uint2 r = make_uint2(0u, 0u);
        if (!done) r = __ldg(bi.tr.base + PrefixTable::off(d) + pair_rev(fkey, d));
        work += work_unit(done ? 1u : 2u);
        if (f.x > f.y || done) {
          have = false;
          if (f.x <= f.y) {
            const unsigned long long rs = atomicAdd(qu.n_raws, 1ull);
            if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{q, f.x, f.y, 1u};
          }
          continue;
        }
        pos += int(tt);
        x = f.x;
        y = f.y;
        zz = r.x;
        ww = r.y;
        sh = false;
      }
      continue;
    }
    const uint32_t sym = pat_sym(pw0, pw1, pos);
    if (!fwd) {  // case A: backward, one symbol
      uint32_t k2, l2;
      if (sh) {
        const uint2 e = __ldg(bi.tf.base + PrefixTable::off(y + 1u) + 4u * x + sym);
        k2 = e.x;
        l2 = e.y;
        work += work_unit(1u);
      } else {
        constexpr uint32_t kC = LineTraits<W>::kChars;
        const uint32_t low = x - 1u;
        const uint32_t jh = line_of<W>(y), jl = line_of<W>(low);
        uint32_t bh[4], bl[4];
        uint64_t wh[W], wl[W];
        load_line<W, 0>(ix, jh, y - jh * kC, bh, wh);
        if (FMG_CHAIN_COND_LOW && jl == jh) {  // same line: no second request
#pragma unroll
          for (int t2 = 0; t2 < 4; ++t2) bl[t2] = bh[t2];
#pragma unroll
          for (int t2 = 0; t2 < W; ++t2) wl[t2] = wh[t2];
        } else {
          load_line<W, 0>(ix, jl, low - jl * kC, bl, wl);
        }
        const uint32_t cs = c_of(ix, sym);
        k2 = cs + occ1_from_line<W>(ix, bl, wl, low, low - jl * kC, sym) + 1u;
        l2 = cs + occ1_from_line<W>(ix, bh, wh, y, y - jh * kC, sym);
        work += work_unit(jl != jh ? 2u : 1u);
      }
      const bool empty = k2 > l2;
      if (empty || pos == 0 || __popcll(dbits & ((1ull << pos) - 1ull)) > 0u) {
        have = false;
        if (!empty && pos == 0) {
          const unsigned long long rs = atomicAdd(qu.n_raws, 1ull);
          if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{q, k2, l2, 1u};
        }
        continue;
      }
      const bool child_sh = sh && y + 1u < K;
      x = child_sh ? sym + 4u * x : k2;
      y = child_sh ? y + 1u : l2;
      sh = child_sh;
      --pos;
      continue;
    }
    // case B: forward, needs all four counts of the reverse index
    uint32_t ck[4], cl[4];
    children4<W>(bi.rev, bi.tr, sh, zz, ww, ck, cl, work);
    const bool dollar = sh ? (zz == bi.tail[ww]) : (zz <= sent_r && sent_r <= ww);
    uint32_t k = x + (dollar ? 1u : 0u);
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b)
      if (b < sym) k += cl[b] + 1u - ck[b];
    const uint32_t sz = sel4(cl, sym) + 1u - sel4(ck, sym);
    if (sz == 0u || pos + 1 == m) {
      have = false;
      if (sz != 0u) {
        const unsigned long long rs = atomicAdd(qu.n_raws, 1ull);
        if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{q, k, k + sz - 1u, 1u};
      }
      continue;
    }
    const bool child_sh = sh && ww + 1u < K;
    zz = child_sh ? sym + 4u * zz : sel4(ck, sym);
    ww = child_sh ? ww + 1u : sel4(cl, sym);
    x = k;
    y = k + sz - 1u;
    sh = child_sh;
    ++pos;
  }
  flush_work(steps, work);
}

// tail[d] = key of the reversed text's first d characters = text[n-1],
// text[n-2], ... (text[n-1] in bits 0..1): BWT[0] = text[n-1] (row 0 is the
// '$' suffix), then one LF step per character (search.py:172-186).
template <int W>
__global__ void k_tail_keys(IndexView ix, uint32_t k, uint32_t* __restrict__ tail) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  uint32_t row = 0, key = 0;
  tail[0] = 0u;
  bool live = true;
  for (uint32_t d = 1; d < 16; ++d) {
    if (live && d <= ix.n && d < k) {
      uint32_t sym;
      const uint32_t prev = psi_step<W>(ix, row, sym);
      key |= sym << (2 * (d - 1));
      tail[d] = key;
      row = prev;
    } else {
      live = false;
      tail[d] = 0xFFFFFFFFu;
    }
  }
}

}  // namespace fmg
