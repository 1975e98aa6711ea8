// Bounded-difference search kernels (search.py:97-159): lower bound, DFS engine,
// level-synchronous z = 1 engine, result sort / dedup / gather.
// Part of libfmgpu.so (sm_100a); included once by fmgpu.cu.
#pragma once

#include <cstdint>
#include "kernels_search.cuh"  // PatternSources
#include "occ_device.cuh"

namespace fmg {

// ----- bounded-difference search -----------------------------------------

// Lower-bound pass of the inexact search as its own kernel (patterns of
// length <= 64): one thread per pattern extends right to left with resets;
// every time W[pos..seg_end] is absent from the text, bit seg_end is set and
// the search restarts from the root at pos-1.  D(i) = popcount of the bits
// <= i (see k_inexact).  Running it apart keeps the DFS kernel's lanes in
// one phase.
template <int W>
__global__ void __launch_bounds__(256) k_dbound(IndexView ix, CodePatterns cp, uint64_t count,
                                                uint64_t* __restrict__ dbits_out, unsigned long long* steps,
                                                PrefixTable pt, const uint2* __restrict__ tx, uint32_t kx) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  uint64_t pw0, pw1;
  int m;
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
  constexpr uint32_t kC = LineTraits<W>::kChars;
  // Table depth: prefix levels 1..pt.k, plus level kx = pt.k + 1 when given.
  const int Kt = pt.base ? int(tx ? kx : pt.k) : 0;
  auto gather = [&](int len, int a) -> uint2 {  // interval of W[a .. a+len-1] (first empty one if absent)
    uint64_t x = pw0, y = pw1;
    const uint32_t sh = uint32_t(2 * a);
    uint64_t lo, mid, hi;  // 128-bit funnel shift (counts >= 64 give 0, see pat_key)
    asm("shr.b64 %0, %1, %2;" : "=l"(lo) : "l"(x), "r"(sh));
    asm("shl.b64 %0, %1, %2;" : "=l"(mid) : "l"(y), "r"(64u - sh));
    asm("shr.b64 %0, %1, %2;" : "=l"(hi) : "l"(y), "r"(sh - 64u));
    const uint32_t key = uint32_t((lo | mid | hi) & ((uint64_t(1) << (2 * len)) - 1u));
    return len > int(pt.k) ? __ldg(tx + key) : __ldg(pt.base + PrefixTable::off(uint32_t(len)) + key);
  };
  uint64_t bits = 0;
  uint64_t work = 0;
  int seg_end = m - 1;
  while (seg_end >= 0) {
    // the run W[pos+1 .. seg_end] is present with interval (k, l); (0, n) = empty run
    uint32_t k = 0, l = ix.n;
    int pos = seg_end;
    if (Kt > 0) {
      // the longest run the tables cover in ONE gather; absent: binary search
      // for the shortest absent suffix (presence is monotone in the length)
      const int L = min(Kt, seg_end + 1);
      const uint2 e = gather(L, seg_end - L + 1);
      work += work_unit(1u);
      if (e.x <= e.y) {
        k = e.x;
        l = e.y;
        pos = seg_end - L;
      } else {
        int lo = 0, hi = L;  // suffix of length lo present, hi absent
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          const uint2 f = gather(mid, seg_end - mid + 1);
          work += work_unit(1u);
          if (f.x <= f.y)
            lo = mid;
          else
            hi = mid;
        }
        bits |= 1ull << seg_end;  // W[seg_end-hi+1 .. seg_end] is absent
        seg_end -= hi;
        continue;
      }
    }
    bool reset = false;
    for (; pos >= 0; --pos) {
      const uint32_t b = uint32_t((pos < 32 ? pw0 : pw1) >> ((pos & 31) << 1)) & 3u;
      const uint32_t cb = c_of(ix, b);
      uint32_t k2, l2;
      if (k == 0u && l == ix.n) {  // root: init_interval, no memory
        k2 = cb + 1u;
        l2 = c_of(ix, b + 1u);
      } else {
        const uint32_t low = k - 1u;
        const uint32_t jh = line_of<W>(l), jl = line_of<W>(low);
        const uint32_t rh = l - jh * kC, rl = low - jl * kC;
        uint32_t bh[4], bl[4];
        uint64_t wh[W], wl[W];
        load_line<W, false>(ix, jh, rh, bh, wh);
        uint32_t ol;
        if (jl != jh) {
          load_line<W, false>(ix, jl, rl, bl, wl);
          ol = occ1_from_line<W>(ix, bl, wl, low, rl, b);
        } else {
          ol = occ1_from_line<W>(ix, bh, wh, low, rl, b);
        }
        k2 = cb + ol + 1u;
        l2 = cb + occ1_from_line<W>(ix, bh, wh, l, rh, b);
        work += work_unit(jl != jh ? 2u : 1u);
      }
      if (k2 > l2) {  // W[pos..seg_end] is absent from the text
        bits |= 1ull << seg_end;
        seg_end = pos - 1;
        reset = true;
        break;
      }
      k = k2;
      l = l2;
    }
    if (!reset) break;  // the run reached the pattern's left end
  }
  dbits_out[q] = bits;
  flush_work(steps, work);
}

// Per-thread global scratch for the inexact engine, warp-blocked (element e
// of lane L of warp w at (w*N + e)*32 + L) so a warp's region is contiguous.
// The DFS stack itself lives in shared memory (see k_inexact).
struct InexactScratch {
  uint4* table;     // H = 2R slots {k, l, epoch, used}: open-addressing dedup of results
  uint32_t* slots;  // R entries: occupied table slots, in insertion order
  uint8_t* dlb;     // Mmax entries: lower bound D[i] (long patterns only)
  uint32_t S, R, Mmax;
  uint64_t T;
  // first pattern of each thread uses epoch0 + 1; every entry already in
  // the table carries an epoch <= epoch0 (EpochTable), so it reads as empty
  uint32_t epoch0;
};

struct InexactOut {
  uint2* kl;          // reserved by atomicAdd on *total
  uint8_t* diffs;
  unsigned long long* total;
  uint64_t cap;
  uint64_t* res_off;  // per pattern: offset in this pass's buffer
  uint32_t* res_cnt;  // per pattern: number of results
  uint8_t* res_pass;  // per pattern: pass that produced it
  uint8_t pass;
  uint32_t* fail_list;  // patterns to retry with larger capacities
  unsigned long long* fail_count;
  unsigned long long* next;  // work-queue cursor
  unsigned long long* steps;
  unsigned long long* unsorted;  // patterns written with > S results (post-sorted)
  uint32_t* unsorted_list;       // their pattern ids (capacity: count)
};

#ifndef FMG_LUT_HINT
#define FMG_LUT_HINT 0  // 1: prefix-table loads with an L2 evict_last policy
#endif
#ifndef FMG_INEX_LINE_HINT
#define FMG_INEX_LINE_HINT 0  // 2: DFS index-line loads with an L2 evict_first policy
#endif

// Reference semantics (search.py:120-159): nodes (i, budget, k, l) from the
// root (m-1, z, 0, n); a node with i < 0 is a result with z - budget diffs;
// otherwise one Occ step at (k-1, l) and children skip (i-1, budget-1, k, l),
// insert (i, budget-1, k', l'), match (i-1, budget, k', l') / mismatch
// (i-1, budget-1, k', l') for every symbol with a non-empty k' <= l'.  The
// set of (interval, min diffs) the DFS reaches does not depend on visiting
// order, so the traversal order is free.
//
// Visiting order: a budget-0 node has only its match child, which is
// continued in registers, so budget-0 chains — most of the steps — never
// touch the stack.  A node with budget >= 1 pushes its match child (same
// budget) first and then its budget-1 children, and the next iteration pops
// the last one; the stack stays budget-monotone — one budget-z entry and at
// most 9 per lower level, depth <= 9z + 1 — small enough for shared memory.
//
// Lower-bound prune (result-preserving): before the DFS, one right-to-left
// exact pass with resets splits W into disjoint segments absent from the
// text; D(i) = number of those segments lying inside W[0..i].  Every way of
// turning W[0..i] into a substring of the text must touch each absent
// segment with its own edit, so a node with D(i) > budget yields nothing and
// is never pushed.  (BWA's D array, computed with the forward index only.)
//
// Shallow nodes (prefix table present): a node whose string S (the text
// characters its path consumed) is shorter than pt.k is held as (key(S), |S|)
// instead of (k, l); its Occ step is one 32-byte table sector giving all four
// child intervals.  Shallow strings are shared by every pattern, so these
// sectors stay in L2, where the index lines of the same wide intervals —
// two random DRAM fetches per step — do not.
template <bool kShort, int W>
__global__ void __launch_bounds__(128) k_inexact(IndexView ix, CodePatterns cp, const uint32_t* __restrict__ list,
                                                 uint64_t count, uint32_t z, InexactScratch sc, InexactOut out,
                                                 PrefixTable pt) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t S = sc.S, nt = blockDim.x, tid = threadIdx.x;
  uint2* s_kl = reinterpret_cast<uint2*>(smem);                     // [S + 1][nt]
  uint32_t* s_ib = reinterpret_cast<uint32_t*>(s_kl + (S + 1) * nt);  // [S + 1][nt]; slot S: push dump
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= sc.T) return;
  uint64_t my_steps = 0;
  const uint64_t wbase = t >> 5, lane = t & 31u;
  auto HI = [&](uint32_t e) -> uint64_t { return (wbase * (2u * sc.R) + e) * 32u + lane; };
  auto LI = [&](uint32_t e) -> uint64_t { return (wbase * sc.R + e) * 32u + lane; };
  uint32_t epoch = sc.epoch0;  // per-thread pattern counter: table slots of older patterns read as empty
  auto DI = [&](uint32_t e) -> uint64_t { return (wbase * sc.Mmax + e) * 32u + lane; };

  // per-pattern state
  bool have = false;
  uint64_t q = 0;
  const uint8_t* codes = nullptr;
  int m = 0;
  uint64_t pw0 = 0, pw1 = 0;  // kShort: the pattern, packed
  uint64_t dbits = 0;         // kShort: right ends of absent segments
  int phase = 0;              // 0: lower-bound pass, 1: DFS
  int pos = 0, seg_end = 0;   // lower-bound pass cursor
  uint32_t kd = 0, ld = 0;    // lower-bound pass interval
  uint32_t sp = 0, nres = 0;
  bool overflow = false;
  bool cur_valid = false;  // DFS node held in registers
  int ci = 0;
  uint32_t cb = 0, ck = 0, cl = 0;  // budget; (k, l), or (key, depth) when csh
  bool csh = false;

  auto sym_at = [&](int i) -> uint32_t {
    if (kShort) return uint32_t((i < 32 ? pw0 : pw1) >> ((i & 31) << 1)) & 3u;
    return uint32_t(__ldg(codes + i));
  };
  auto dlb = [&](int i) -> uint32_t {
    if (kShort) return __popcll(dbits & ((2ull << i) - 1ull));
    return sc.dlb[DI(uint32_t(i))];
  };
  // best[(k, l)] = min used (search.py:127-134) in a per-thread hash table
  auto record = [&](uint32_t k, uint32_t l, uint32_t used) {
    const uint32_t H = 2u * sc.R;
    uint32_t h = (k * 0x9E3779B1u ^ l * 0x85EBCA77u) & (H - 1u);
    for (uint32_t probe = 0; probe < H; ++probe, h = (h + 1u) & (H - 1u)) {
      uint4 e = sc.table[HI(h)];
      if (e.z != epoch) {  // empty for this pattern: insert
        if (nres == sc.R) {
          overflow = true;
          return;
        }
        sc.table[HI(h)] = make_uint4(k, l, epoch, used);
        sc.slots[LI(nres)] = h;
        ++nres;
        return;
      }
      if (e.x == k && e.y == l) {
        if (used < e.w) sc.table[HI(h)].w = used;
        return;
      }
    }
    overflow = true;
  };
  auto fail = [&]() {
    const unsigned long long f = atomicAdd(out.fail_count, 1ull);
    out.fail_list[f] = uint32_t(q);
    out.res_cnt[q] = 0;
  };
  auto finish = [&]() {
    if (overflow) {
      fail();
      return;
    }
    uint64_t o = 0;
    if (nres) {
      o = atomicAdd(out.total, (unsigned long long)nres);
      if (o + nres > out.cap) {  // this pass's buffer is full: retry later
        fail();
        return;
      }
      if (nres <= S) {
        // The DFS stack is empty now: reuse this thread's shared-memory stack
        // slots to insertion-sort the results by (k, l) (unique after dedup).
        for (uint32_t r = 0; r < nres; ++r) {
          const uint4 e = sc.table[HI(sc.slots[LI(r)])];
          uint32_t b = r;
          while (b > 0) {
            const uint2 p = s_kl[(b - 1) * nt + tid];
            if (p.x < e.x || (p.x == e.x && p.y < e.y)) break;
            s_kl[b * nt + tid] = p;
            s_ib[b * nt + tid] = s_ib[(b - 1) * nt + tid];
            --b;
          }
          s_kl[b * nt + tid] = make_uint2(e.x, e.y);
          s_ib[b * nt + tid] = e.w;
        }
        for (uint32_t r = 0; r < nres; ++r) {
          out.kl[o + r] = s_kl[r * nt + tid];
          out.diffs[o + r] = uint8_t(s_ib[r * nt + tid]);
        }
      } else {  // unsorted; the host runs a segmented sort afterwards
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

  while (true) {
    // ---- acquire the next node that needs an Occ step ----
    uint32_t k = 0, l = 0;
    bool stepping = false;
    while (!stepping) {
      if (!have) {
        // persistent work queue: one atomic per pattern balances the
        // per-pattern DFS sizes across lanes and SMs
        const unsigned long long slot = atomicAdd(out.next, 1ull);
        if (slot >= count) break;
        q = list ? list[slot] : slot;
        if (kShort && cp.packed1) {  // caller-packed fixed-length patterns
          m = int(cp.fixed_m);
          pw0 = cp.packed1[q];
          pw1 = 0;
          dbits = cp.dbits ? cp.dbits[q] : 0ull;
        } else if (kShort) {
          m = int(cp.offsets[q + 1] - cp.offsets[q]);
          const ulonglong2 pk = cp.packed[q];
          pw0 = pk.x;
          pw1 = pk.y;
          dbits = cp.dbits ? cp.dbits[q] : 0ull;
        } else {
          const uint64_t o0 = cp.offsets[q], o1 = cp.offsets[q + 1];
          codes = cp.codes + o0;
          m = int(o1 - o0);
          for (int j = 0; j < m; ++j) sc.dlb[DI(uint32_t(j))] = 0;
        }
        phase = 0;
        pos = m - 1;
        seg_end = m - 1;
        kd = 0;  // the pass starts from the root interval [0, n]
        ld = ix.n;
        if (kShort && cp.dbits) pos = -1;  // lower bound precomputed by k_dbound
        sp = nres = 0;
        ++epoch;
        overflow = false;
        cur_valid = false;
        have = true;
      }
      if (phase == 0) {
        if (pos < 0) {
          if (!kShort) {  // flags of segment ends -> D(i) = ends at or before i
            uint32_t acc = 0;
            for (int j = 0; j < m; ++j) {
              uint8_t* d = &sc.dlb[DI(uint32_t(j))];
              acc += *d;
              *d = uint8_t(min(acc, 255u));
            }
          }
          phase = 1;
          // root (search.py:125), held in registers
          cur_valid = dlb(m - 1) <= z;
          ci = m - 1;
          cb = z;
          csh = pt.base != nullptr;  // the root's string is empty: key 0, depth 0
          ck = 0u;
          cl = csh ? 0u : ix.n;
          continue;
        }
        k = kd;
        l = ld;
        stepping = true;
      } else {
        if (overflow) {
          finish();
          have = false;
          continue;
        }
        if (!cur_valid) {
          if (sp == 0) {
            finish();
            have = false;
            continue;
          }
          --sp;
          const uint2 e = s_kl[sp * nt + tid];
          const uint32_t ib = s_ib[sp * nt + tid];
          ci = int(ib >> 16) - 1;
          cb = ib & 0xFFu;
          csh = (ib >> 15) & 1u;
          ck = e.x;
          cl = e.y;
          cur_valid = true;
        }
        k = ck;
        l = cl;
        stepping = true;
      }
    }
    if (!stepping) break;

    // ---- one Occ step: the four child intervals of (k, l) ----
    uint32_t k2[4], l2[4];
    if (phase == 1 && csh) {  // shallow node: one prefix-table sector
      const uint2* p = pt.base + PrefixTable::off(l + 1u) + 4u * k;
      uint64_t a0, a1, a2, a3;
#if FMG_LUT_HINT
      uint64_t pol;
      asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      asm("ld.global.nc.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
          : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
          : "l"(p), "l"(pol));
#else
      ld256<0>(reinterpret_cast<const uint8_t*>(p), a0, a1, a2, a3);
#endif
      k2[0] = uint32_t(a0), l2[0] = uint32_t(a0 >> 32), k2[1] = uint32_t(a1), l2[1] = uint32_t(a1 >> 32);
      k2[2] = uint32_t(a2), l2[2] = uint32_t(a2 >> 32), k2[3] = uint32_t(a3), l2[3] = uint32_t(a3 >> 32);
      my_steps += work_unit(1u);
    } else {
      uint32_t lo[4], hi[4];
      my_steps += work_unit(occ_step<W, FMG_INEX_LINE_HINT>(ix, k, l, lo, hi));
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        k2[b] = ix.c[b] + lo[b] + 1u;
        l2[b] = ix.c[b] + hi[b];
      }
    }

    if (phase == 0) {
      const uint32_t b = sym_at(pos);
      const uint32_t kb = sel4(k2, b), lb = sel4(l2, b);
      if (kb > lb) {  // W[pos..seg_end] is absent from the text
        if (kShort)
          dbits |= 1ull << seg_end;
        else
          sc.dlb[DI(uint32_t(seg_end))] = 1;
        kd = 0;
        ld = ix.n;
        seg_end = pos - 1;
      } else {
        kd = kb;
        ld = lb;
      }
      --pos;
      continue;
    }

    // ---- DFS expansion of the register node (search.py:135-152) ----
    const int i = ci;
    const uint32_t budget = cb;
    const uint32_t want = sym_at(i);
    const uint32_t kw = sel4(k2, want), lw = sel4(l2, want);
    // children stay shallow while their strings are shorter than pt.k
    const bool child_sh = csh && cl + 1u < pt.k;
    if (budget == 0) {
      // budget-0 node: only the match child, continued in registers
      if (kw > lw) {
        cur_valid = false;
      } else if (i == 0) {
        record(kw, lw, z);
        cur_valid = false;
      } else {
        ci = i - 1;
        ck = child_sh ? want + 4u * ck : kw;
        cl = child_sh ? cl + 1u : lw;
        csh = child_sh;
        cur_valid = dlb(i - 1) == 0;
      }
      continue;
    }
    // budget >= 1: push every viable child with predicated stores (match
    // child first, so it is popped last), then pop the top as the continue
    // node.  Straight-line code: a lane expanding such a node costs its warp
    // little more than a budget-0 step.
    const uint32_t bm1 = budget - 1u;
    const bool at0 = i == 0;
    const uint32_t d_prev = at0 ? 0u : dlb(i - 1), d_cur = dlb(i);
    const bool ok_match = !at0 && d_prev <= budget;  // (i-1, budget)
    const bool ok_prev = !at0 && d_prev <= bm1;      // skip / mismatch: (i-1, budget-1)
    const bool ok_cur = d_cur <= bm1;                // insert: (i, budget-1)
    if (at0) {  // children with i - 1 < 0 are results (rare)
      if (kw <= lw) record(kw, lw, z - budget);
      uint32_t sk = ck, sl = cl;  // skip: this node's own interval
      if (csh) {
        if (cl == 0u) {
          sk = 0u;
          sl = ix.n;
        } else {
          const uint2 e = __ldg(pt.base + PrefixTable::off(cl) + ck);
          sk = e.x;
          sl = e.y;
        }
      }
      record(sk, sl, z - bm1);
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (b != want && k2[b] <= l2[b]) record(k2[b], l2[b], z - bm1);  // mismatch
    }
    // Branch-free push: every candidate is stored, a rejected one into the
    // dump slot S (the stack has S + 1 entries), and sp advances by `ok`.
    auto push_if = [&](bool cond, int pi, uint32_t pb, uint32_t pk, uint32_t pl, bool psh) {
      const bool ok = cond && sp < S;
      overflow |= cond && sp >= S;
      const uint32_t slot = ok ? sp : S;
      s_kl[slot * nt + tid] = make_uint2(pk, pl);
      s_ib[slot * nt + tid] = (uint32_t(pi + 1) << 16) | (psh ? 0x8000u : 0u) | pb;
      sp += ok ? 1u : 0u;
    };
    const uint32_t ckey = 4u * ck, cdep = cl + 1u;  // shallow children: key b + 4 key(S), depth + 1
    push_if(ok_match && kw <= lw, i - 1, budget, child_sh ? want + ckey : kw, child_sh ? cdep : lw,
            child_sh);                                  // match
    push_if(ok_prev, i - 1, bm1, ck, cl, csh);           // skip: same string
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b) {
      const bool ne = k2[b] <= l2[b];
      const uint32_t px = child_sh ? b + ckey : k2[b], py = child_sh ? cdep : l2[b];
      push_if(ok_cur && ne, i, bm1, px, py, child_sh);                 // insert
      push_if(ok_prev && ne && b != want, i - 1, bm1, px, py, child_sh);  // mismatch
    }
    cur_valid = false;  // the next iteration pops the top (the last child pushed)
  }
  flush_work(out.steps, my_steps);
}

// Sort the results of patterns that had more than S of them (written
// unsorted by k_inexact) in place: one block per pattern, bitonic sort of
// (k << 32 | l, diffs) in shared memory.  Segments above kSortMax entries set
// *too_big and the host falls back to a CUB segmented sort.
constexpr uint32_t kSortMax = 4096;
__global__ void __launch_bounds__(256) k_sort_segments(const uint32_t* __restrict__ list, const uint64_t* __restrict__ res_off,
                                                       const uint32_t* __restrict__ res_cnt, uint2* __restrict__ kl,
                                                       uint8_t* __restrict__ diffs, uint32_t* __restrict__ too_big) {
  __shared__ uint64_t key[kSortMax];
  __shared__ uint8_t val[kSortMax];
  const uint32_t q = list[blockIdx.x];
  const uint32_t n = res_cnt[q];
  const uint64_t o = res_off[q];
  if (n > kSortMax) {
    if (threadIdx.x == 0) atomicOr(too_big, 1u);
    return;
  }
  uint32_t p = 1;
  while (p < n) p <<= 1;
  for (uint32_t j = threadIdx.x; j < p; j += blockDim.x) {
    if (j < n) {
      const uint2 e = kl[o + j];
      key[j] = (uint64_t(e.x) << 32) | e.y;
      val[j] = diffs[o + j];
    } else {
      key[j] = ~0ull;
      val[j] = 0;
    }
  }
  __syncthreads();
  for (uint32_t size = 2; size <= p; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t j = threadIdx.x; j < p; j += blockDim.x) {
        const uint32_t partner = j ^ stride;
        if (partner > j) {
          const bool up = (j & size) == 0;
          const uint64_t a = key[j], b = key[partner];
          if ((a > b) == up) {
            key[j] = b;
            key[partner] = a;
            const uint8_t t = val[j];
            val[j] = val[partner];
            val[partner] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
    kl[o + j] = make_uint2(uint32_t(key[j] >> 32), uint32_t(key[j]));
    diffs[o + j] = val[j];
  }
}

// ----- level-synchronous engine for z = 1 ----------------------------------
//
// For a budget of one edit the DFS of search.py:120-159 decomposes into (a)
// the exact "spine" walk of budget-1 match children from the root and (b)
// independent budget-0 continuations spawned at every spine node — skip,
// inserts, mismatches — each of which is an exact backward search of the
// remaining prefix from its own interval.  k_spine walks every spine and
// queues the continuations; k_chain walks every continuation; both emit raw
// (pattern, k, l, diffs) results, deduplicated and sorted per pattern
// afterwards.  Every lane of a warp runs the same loop, which the DFS kernel
// cannot offer.  The reached (interval, min diffs) set equals the DFS's.

struct Z1Node {  // a budget-0 continuation: pattern q, next position i, interval
  uint32_t q, i, k, l;
};
struct Z1Raw {  // one reached result before dedup
  uint32_t q, k, l, used;
};
struct Z1Queues {
  Z1Node* nodes;
  unsigned long long* n_nodes;
  uint64_t node_cap;
  Z1Raw* raws;
  unsigned long long* n_raws;
  uint64_t raw_cap;
};

// Warp-aggregated append of `cnt` (0..15) slots: one atomic per warp.
__device__ __forceinline__ uint64_t warp_reserve(unsigned long long* counter, uint32_t cnt) {
  const unsigned mask = __activemask();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t prefix = 0, total = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const unsigned bal = __ballot_sync(mask, (cnt >> b) & 1u);
    prefix += uint32_t(__popc(bal & lt)) << b;
    total += uint32_t(__popc(bal)) << b;
  }
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (int(lane) == leader && total) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(mask, base, leader);
  return base + prefix;
}

__device__ __forceinline__ void z1_pattern(const CodePatterns& cp, uint64_t q, uint64_t& pw0, uint64_t& pw1, int& m) {
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

__device__ __forceinline__ uint32_t z1_sym(uint64_t pw0, uint64_t pw1, int i) {
  return uint32_t((i < 32 ? pw0 : pw1) >> ((i & 31) << 1)) & 3u;
}

__device__ __forceinline__ uint32_t z1_dlb(uint64_t dbits, int i) { return __popcll(dbits & ((2ull << i) - 1ull)); }

template <int W>
__global__ void __launch_bounds__(256) k_spine(IndexView ix, CodePatterns cp, uint64_t count, Z1Queues qu,
                                               unsigned long long* steps) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  uint64_t pw0, pw1;
  int m;
  z1_pattern(cp, q, pw0, pw1, m);
  const uint64_t dbits = cp.dbits[q];
  uint64_t my_steps = 0;
  int i = m - 1;
  uint32_t k = 0, l = ix.n;
  bool alive = z1_dlb(dbits, m - 1) <= 1u;  // root (m-1, 1, 0, n), search.py:125
  while (alive) {
    uint32_t lo[4], hi[4];
    my_steps += work_unit(occ_step<W, false>(ix, k, l, lo, hi));
    const uint32_t want = z1_sym(pw0, pw1, i);
    uint32_t k2[4], l2[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      k2[b] = ix.c[b] + lo[b] + 1u;
      l2[b] = ix.c[b] + hi[b];
    }
    const bool at0 = i == 0;
    const bool ok_prev = !at0 && z1_dlb(dbits, i - 1) == 0u;  // (i-1, budget 0)
    const bool ok_cur = z1_dlb(dbits, i) == 0u;               // (i, budget 0)
    // budget-0 children to queue: skip, 4 inserts, 3 mismatches
    bool e[8];
    e[0] = ok_prev;  // skip (i-1, 0, k, l)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const bool ne = k2[b] <= l2[b];
      e[1 + b] = ok_cur && ne;  // insert (i, 0, k_b, l_b)
    }
    uint32_t mm = 0;  // mismatch slots 5..7 hold the three b != want in order
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (uint32_t(b) == want) continue;
      e[5 + mm] = ok_prev && (k2[b] <= l2[b]);
      ++mm;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) cnt += e[j] ? 1u : 0u;
    uint64_t slot = warp_reserve(qu.n_nodes, cnt);
    auto put = [&](uint32_t ni, uint32_t nk, uint32_t nl) {
      if (slot < qu.node_cap) qu.nodes[slot] = Z1Node{uint32_t(q), ni, nk, nl};
      ++slot;
    };
    if (e[0]) put(uint32_t(i - 1), k, l);
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (e[1 + b]) put(uint32_t(i), k2[b], l2[b]);
    mm = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (uint32_t(b) == want) continue;
      if (e[5 + mm]) put(uint32_t(i - 1), k2[b], l2[b]);
      ++mm;
    }
    // children with i - 1 < 0 are results (search.py:127-134): rare
    uint32_t rc = 0;
    if (at0) {
      rc = 1u;  // skip
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (uint32_t(b) != want && k2[b] <= l2[b]) ++rc;
      if (sel4(k2, want) <= sel4(l2, want)) ++rc;  // match with budget kept
    }
    uint64_t rs = warp_reserve(qu.n_raws, rc);
    if (at0) {
      auto rput = [&](uint32_t rk, uint32_t rl, uint32_t used) {
        if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{uint32_t(q), rk, rl, used};
        ++rs;
      };
      rput(k, l, 1u);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (uint32_t(b) != want && k2[b] <= l2[b]) rput(k2[b], l2[b], 1u);
      if (sel4(k2, want) <= sel4(l2, want)) rput(sel4(k2, want), sel4(l2, want), 0u);
      break;
    }
    // continue along the match child (i-1, 1)
    const uint32_t kw = sel4(k2, want), lw = sel4(l2, want);
    if (kw > lw || z1_dlb(dbits, i - 1) > 1u) break;
    k = kw;
    l = lw;
    --i;
  }
  flush_work(steps, my_steps);
}

template <int W>
__global__ void __launch_bounds__(256) k_chain(IndexView ix, CodePatterns cp, const Z1Node* __restrict__ nodes,
                                               uint64_t n_nodes, Z1Queues qu, unsigned long long* steps) {
  // Persistent grid, lane refill: most continuations die within a few steps
  // while the few that match run to i < 0, so a lane takes its next node as
  // soon as its chain ends instead of idling until its warp's longest chain.
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t my_steps = 0;
  uint64_t pw0 = 0, pw1 = 0, dbits = 0;
  int i = -1;
  uint32_t k = 0, l = 0, q = 0;
  bool have = false;
  while (true) {
    if (!have) {
      if (t >= n_nodes) break;
      const Z1Node nd = nodes[t];
      t += stride;
      int m;
      z1_pattern(cp, nd.q, pw0, pw1, m);
      dbits = cp.dbits[nd.q];
      q = nd.q;
      i = int(nd.i);
      k = nd.k;
      l = nd.l;
      have = true;
    }
    // budget-0 node (i, k, l): only its match child
    const uint32_t sym = z1_sym(pw0, pw1, i);
    uint32_t k2, l2;
    if (k == 0u && l == ix.n) {
      k2 = c_of(ix, sym) + 1u;
      l2 = c_of(ix, sym + 1u);
    } else {
      const uint32_t low = k - 1u;
      const uint32_t jh = line_of<W>(l), jl = line_of<W>(low);
      const uint32_t rh = l - jh * kC, rl = low - jl * kC;
      uint32_t bh[4], bl[4];
      uint64_t wh[W], wl[W];
      load_line<W, false>(ix, jh, rh, bh, wh);
      uint32_t ol;
      if (jl != jh) {
        load_line<W, false>(ix, jl, rl, bl, wl);
        ol = occ1_from_line<W>(ix, bl, wl, low, rl, sym);
      } else {
        ol = occ1_from_line<W>(ix, bh, wh, low, rl, sym);
      }
      const uint32_t cs = c_of(ix, sym);
      k2 = cs + ol + 1u;
      l2 = cs + occ1_from_line<W>(ix, bh, wh, l, rh, sym);
      my_steps += work_unit(jl != jh ? 2u : 1u);
    }
    const bool empty = k2 > l2;
    const bool found = !empty && i == 0;
    if (empty || found || z1_dlb(dbits, i - 1) > 0u) {
      have = false;
      if (found) {
        const unsigned long long rs = atomicAdd(qu.n_raws, 1ull);
        if (rs < qu.raw_cap) qu.raws[rs] = Z1Raw{q, k2, l2, 1u};
      }
      continue;
    }
    k = k2;
    l = l2;
    --i;
  }
  flush_work(steps, my_steps);
}

// counting sort of raw results by pattern
__global__ void k_z1_hist(const Z1Raw* __restrict__ raws, uint64_t n, uint32_t* __restrict__ per_q) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) atomicAdd(&per_q[raws[t].q], 1u);
}

__global__ void k_z1_scatter(const Z1Raw* __restrict__ raws, uint64_t n, uint64_t* __restrict__ cursor,
                             uint64_t* __restrict__ keys, uint8_t* __restrict__ used) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Z1Raw r = raws[t];
  const unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[r.q]), 1ull);
  keys[p] = (uint64_t(r.k) << 32) | r.l;
  used[p] = uint8_t(r.used);
}

// per pattern: unique (k, l) with min diffs over its sorted segment
__global__ void k_z1_unique_count(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ used,
                                  const uint64_t* __restrict__ seg, uint64_t count, uint32_t* __restrict__ ucnt) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  uint32_t c = 0;
  for (uint64_t j = seg[q]; j < seg[q + 1]; ++j)
    if (j == seg[q] || keys[j] != keys[j - 1]) ++c;
  ucnt[q] = c;
}

__global__ void k_z1_unique_write(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ used,
                                  const uint64_t* __restrict__ seg, const uint64_t* __restrict__ row_off,
                                  uint64_t count, uint32_t* __restrict__ k_out, uint32_t* __restrict__ l_out,
                                  uint8_t* __restrict__ d_out) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  uint64_t o = row_off[q];
  for (uint64_t j = seg[q]; j < seg[q + 1];) {
    const uint64_t key = keys[j];
    uint8_t best = used[j];
    uint64_t e = j + 1;
    for (; e < seg[q + 1] && keys[e] == key; ++e) best = min(best, used[e]);
    k_out[o] = uint32_t(key >> 32);
    l_out[o] = uint32_t(key);
    d_out[o] = best;
    ++o;
    j = e;
  }
}

// Gather per-pattern results of one pass into the final CSR arrays.
__global__ void k_gather_matches(uint64_t count, const uint64_t* __restrict__ res_off,
                                 const uint32_t* __restrict__ res_cnt, const uint8_t* __restrict__ res_pass,
                                 uint8_t pass, const uint2* __restrict__ src_kl, const uint8_t* __restrict__ src_d,
                                 const uint64_t* __restrict__ row_off, uint32_t* __restrict__ k_out,
                                 uint32_t* __restrict__ l_out, uint8_t* __restrict__ d_out) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count || res_pass[q] != pass) return;
  const uint32_t n = res_cnt[q];
  const uint64_t s = res_off[q], d = row_off[q];
  for (uint32_t r = 0; r < n; ++r) {
    const uint2 e = src_kl[s + r];
    k_out[d + r] = e.x;
    l_out[d + r] = e.y;
    d_out[d + r] = src_d[s + r];
  }
}

// 2-bit packing of patterns of length <= 64 for k_inexact (one coalesced-ish
// pass so the search kernel starts a pattern with a single 16-byte load).
__global__ void k_pack_patterns(const uint8_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                                uint64_t count, ulonglong2* __restrict__ packed) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint64_t a = offsets[q], b = offsets[q + 1];
  uint64_t w0 = 0, w1 = 0;
  for (uint64_t j = a; j < b && j < a + 64; ++j) {
    const uint32_t f = uint32_t(j - a);
    const uint64_t v = uint64_t(codes[j] & 3u) << ((f & 31u) << 1);
    if (f < 32u)
      w0 |= v;
    else
      w1 |= v;
  }
  packed[q] = make_ulonglong2(w0, w1);
}

// Pattern batch validation on the device: offsets[0] == 0, every pattern
// non-empty (search.py:83-84), codes in [0, 4); also the longest pattern.
__global__ void k_check_patterns(const uint8_t* __restrict__ codes, const uint64_t* __restrict__ offsets,
                                 uint64_t count, unsigned long long* __restrict__ max_len,
                                 uint32_t* __restrict__ err) {
  // One thread per pattern for the offsets, a grid-stride scan of the code
  // bytes in 8-byte words, and one atomic per warp (a per-thread atomicMax
  // on one address serialised 1M patterns into 660 us on B200).
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  uint32_t len = 0, flags = 0;
  if (q < count) {
    const uint64_t a = offsets[q], b = offsets[q + 1];
    if (q == 0 && a != 0) flags |= 4u;
    if (b <= a) flags |= 1u;
    else len = uint32_t(b - a > 0xFFFFFFFFull ? 0xFFFFFFFFull : b - a);
  }
  // codes[0 .. total) when offsets[0] == 0 (otherwise that error is
  // reported and the codes are not scanned)
  const uint64_t total = offsets[0] == 0 ? offsets[count] : 0;
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(codes) & 7u) == 0) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(codes);
    for (uint64_t i = q; i < total / 8; i += nthreads)
      if (__ldg(w + i) & 0xFCFCFCFCFCFCFCFCull) flags |= 2u;  // a byte > 3
    for (uint64_t j = total / 8 * 8 + q; j < total; j += nthreads)
      if (codes[j] > 3) flags |= 2u;
  } else {
    for (uint64_t j = q; j < total; j += nthreads)
      if (codes[j] > 3) flags |= 2u;
  }
  const uint32_t wl = __reduce_max_sync(0xFFFFFFFFu, len);
  const uint32_t wf = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0) {
    if (wl) atomicMax(max_len, (unsigned long long)wl);
    if (wf) atomicOr(err, wf);
  }
}

__global__ void k_pack_keys(uint64_t n, const uint32_t* __restrict__ k, const uint32_t* __restrict__ l,
                            uint64_t* __restrict__ keys) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (uint64_t(k[i]) << 32) | l[i];
}

__global__ void k_unpack_keys(uint64_t n, const uint64_t* __restrict__ keys, const uint8_t* __restrict__ d_in,
                              uint32_t* __restrict__ k, uint32_t* __restrict__ l, uint8_t* __restrict__ d_out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    k[i] = uint32_t(keys[i] >> 32);
    l[i] = uint32_t(keys[i]);
    d_out[i] = d_in[i];
  }
}

// ---- host-sync-free result collection (run_z1b): sizes come from device
// counters, every kernel is grid-stride, the dedup sort runs per pattern ----

__global__ void k_z1_hist_dev(const Z1Raw* __restrict__ raws, const unsigned long long* __restrict__ n_raw,
                              uint64_t cap, uint32_t* __restrict__ per_q) {
  const uint64_t n = min(uint64_t(*n_raw), cap);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride)
    atomicAdd(&per_q[raws[t].q], 1u);
}

__global__ void k_z1_scatter_dev(const Z1Raw* __restrict__ raws, const unsigned long long* __restrict__ n_raw,
                                 uint64_t cap, uint64_t* __restrict__ cursor, uint64_t* __restrict__ keys,
                                 uint8_t* __restrict__ used) {
  const uint64_t n = min(uint64_t(*n_raw), cap);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
    const Z1Raw r = raws[t];
    const unsigned long long p = atomicAdd(reinterpret_cast<unsigned long long*>(&cursor[r.q]), 1ull);
    keys[p] = (uint64_t(r.k) << 32) | r.l;
    used[p] = uint8_t(r.used);
  }
}

// Per pattern: sort its raw results by (k, l, diffs) in place (insertion
// sort: segments hold a handful of entries), then keep the first of each
// (k, l) — the smallest diffs — compacted at the segment start
// (search.py:128-134, 153-159).  ucnt[q] = the unique count.
__global__ void k_z1_sort_unique(uint64_t* __restrict__ keys, uint8_t* __restrict__ used,
                                 const uint64_t* __restrict__ seg, uint64_t count, uint32_t* __restrict__ ucnt) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint64_t a = seg[q], b = seg[q + 1];
  for (uint64_t i = a + 1; i < b; ++i) {
    const uint64_t kk = keys[i];
    const uint8_t uu = used[i];
    uint64_t j = i;
    while (j > a && (keys[j - 1] > kk || (keys[j - 1] == kk && used[j - 1] > uu))) {
      keys[j] = keys[j - 1];
      used[j] = used[j - 1];
      --j;
    }
    keys[j] = kk;
    used[j] = uu;
  }
  uint32_t c = 0;
  for (uint64_t i = a; i < b; ++i) {
    if (i == a || keys[i] != keys[i - 1]) {
      keys[a + c] = keys[i];
      used[a + c] = used[i];
      ++c;
    }
  }
  ucnt[q] = c;
}

// Unique results of pattern q to their CSR rows (k | l packed in one u64).
__global__ void k_z1_write_kl(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ used,
                              const uint64_t* __restrict__ seg, const uint64_t* __restrict__ row_off, uint64_t count,
                              uint64_t* __restrict__ kl_out, uint8_t* __restrict__ d_out) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint64_t a = seg[q], o = row_off[q], c = row_off[q + 1] - o;
  for (uint64_t i = 0; i < c; ++i) {
    kl_out[o + i] = keys[a + i];
    d_out[o + i] = used[a + i];
  }
}

// k | l packed results -> separate k and l arrays (fmg_matches_copy).
__global__ void k_split_kl(const uint64_t* __restrict__ kl, uint64_t n, uint32_t* __restrict__ k,
                           uint32_t* __restrict__ l) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
    const uint64_t v = kl[t];
    if (k) k[t] = uint32_t(v >> 32);
    if (l) l[t] = uint32_t(v);
  }
}

__global__ void k_widen_counts(uint64_t count, const uint32_t* __restrict__ c32, uint64_t* __restrict__ c64) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < count) c64[q] = c32[q];
}

}  // namespace fmg
