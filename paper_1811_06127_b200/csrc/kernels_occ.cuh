// Index re-layout and Occ-step kernels (occ.py:59-96, index.py:24-36).
// Part of libfmgpu.so (sm_100a); included once by fmgpu.cu.
#pragma once

#include <cstdint>

#include "occ_device.cuh"

namespace fmg {

// Counts of A, C, G, T among all 32 fields of one packed word.
__device__ __forceinline__ void add_word_counts(uint64_t w, uint32_t c[4]) {
  const uint64_t lo = w & kFieldLo, hi = (w >> 1) & kFieldLo;
  const uint32_t t = __popcll(lo & hi), h = __popcll(hi), l = __popcll(lo);
  c[3] += t;
  c[2] += h - t;
  c[1] += l - t;
  c[0] += 32u - h - l + t;
}

// Bucket records (4 x u64 LE base + 32 B chars, 128 chars each) -> lines of
// 32W chars.  Line j starts at char 32Wj, which is a multiple of 32 and so
// falls on a word boundary of its bucket; its checkpoint is the bucket base
// plus the counts of the bucket's words before it.
template <int W>
__global__ void k_build_lines(const uint64_t* __restrict__ rec, uint64_t nb, uint8_t* __restrict__ lines,
                              uint64_t n_lines, uint32_t* __restrict__ err) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n_lines) return;
  const uint64_t c0 = j * LineTraits<W>::kChars;
  const uint64_t b0 = c0 >> 7;
  const uint64_t* r = rec + b0 * 8;
  uint32_t base[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (r[s] >= 0xFFFFFFFFull) atomicOr(err, 1u);
    base[s] = uint32_t(r[s]);
  }
  const uint32_t skip = uint32_t((c0 & 127u) >> 5);
  for (uint32_t q = 0; q < skip; ++q) add_word_counts(r[4 + q], base);
  Line<W> out;
#pragma unroll
  for (int s = 0; s < 4; ++s) out.base[s] = base[s];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const uint64_t c = c0 + 32u * k;
    const uint64_t b = c >> 7;
    out.w[k] = (b < nb) ? rec[b * 8 + 4 + ((c & 127u) >> 5)] : 0ull;
  }
  reinterpret_cast<Line<W>*>(lines)[j] = out;
}

// L2 eviction policies: streamed query/result bytes are marked evict-first
// so they do not push index lines out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint2 ld_stream_u2(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y)
      : "l"(p), "l"(policy_evict_first()));
  return v;
}

__device__ __forceinline__ void st_stream_256(uint32_t* p, const uint32_t lo[4], const uint32_t hi[4]) {
  const uint64_t a = uint64_t(lo[0]) | (uint64_t(lo[1]) << 32);
  const uint64_t b = uint64_t(lo[2]) | (uint64_t(lo[3]) << 32);
  const uint64_t c = uint64_t(hi[0]) | (uint64_t(hi[1]) << 32);
  const uint64_t d = uint64_t(hi[2]) | (uint64_t(hi[3]) << 32);
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "l"(a),
               "l"(b), "l"(c), "l"(d), "l"(policy_evict_first())
               : "memory");
}

// Occ step microkernel.  Thread handles PER pairs strided by blockDim so the
// (k,l) loads and the 32-byte output stores stay fully coalesced; all line
// loads of a thread are issued before any popcount so each thread keeps up
// to 2*PER independent line reads in flight.
//
// kBulk (PER = 1): the block's counts are staged in shared memory and leave
// as ONE bulk copy (cp.async.bulk shared -> global, the TMA path) instead of a
// 32-byte store per thread through the LSU: 89.2 -> 90.6 G steps/s on config
// 1.  (ncu shows the SM's L1 -> crossbar request port 87 % busy before and 89 %
// after, so the bulk copy's payload shares that port with the line requests;
// the gain is the LSU work saved.)
//
// kExch (PER = 1, W = 2): neighbouring lanes fetch for each other so that the
// two lines of ONE step are requested by one instruction — the even lane asks
// for the high line and the odd lane for the low line of the even lane's
// step, then the same for the odd lane's step — and swap the data by shuffle.
// Lines of one step usually share a 128-byte block, which the coalescer turns
// into one L1 -> crossbar request (1.36 requests per config-1 step instead of
// 1.75) without doubling the threads as k_occ_pair_2l does.
#ifndef FMG_OCC_MINB
#define FMG_OCC_MINB 1  // resident 256-thread blocks per SM the register budget is sized for (A/B: 8 = 32 registers)
#endif
template <int PER, int W, bool kBulk = false, bool kExch = false>
__global__ void __launch_bounds__(256, FMG_OCC_MINB) k_occ_pair(IndexView ix, const uint2* __restrict__ kl, uint64_t count,
                                                  uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  static_assert(!kBulk || PER == 1, "the bulk-store form handles one pair per thread");
  static_assert(!kExch || (PER == 1 && W == 2), "the lane-exchange form: one pair per thread, 32-byte lines");
  __shared__ __align__(128) uint32_t stage[kBulk ? 256 * 8 : 4];
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint64_t first = uint64_t(blockIdx.x) * blockDim.x * PER + threadIdx.x;
  uint2 q[PER];
  bool act[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const uint64_t i = first + uint64_t(u) * blockDim.x;
    act[u] = i < count;
    q[u] = act[u] ? ld_stream_u2(kl + i) : make_uint2(1u, 0u);
  }
  uint32_t bh[PER][4], bl[PER][4];
  uint64_t wh[PER][W], wl[PER][W];
  bool ok[PER], two[PER];
  uint32_t rh[PER], rl[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const uint32_t k = q[u].x, l = q[u].y;
    ok[u] = act[u] && l <= ix.n && k <= l + 1u;
    if (act[u] && !ok[u] && err) atomicOr(err, 1u);
    const uint32_t hh = ok[u] ? l : 0u;
    const uint32_t ll = (ok[u] && k != 0u) ? k - 1u : hh;
    const uint32_t jh = line_of<W>(hh), jl = line_of<W>(ll);
    rh[u] = hh - jh * kC;
    rl[u] = ll - jl * kC;
    two[u] = jl != jh;
    if constexpr (kExch) {
      const bool odd = threadIdx.x & 1u;
      const uint32_t jh_p = __shfl_xor_sync(0xFFFFFFFFu, jh, 1), jl_p = __shfl_xor_sync(0xFFFFFFFFu, jl, 1);
      // instruction A: the even lane's step (even: its high line, odd: the partner's low line);
      // instruction B: the odd lane's step (even: the partner's high line, odd: its low line)
      const uint32_t ja = odd ? jl_p : jh, jb = odd ? jl : jh_p;
      uint64_t a[4], b[4];
      ld256<1>(ix.lines + size_t(ja) * 32u, a[0], a[1], a[2], a[3]);
      ld256<1>(ix.lines + size_t(jb) * 32u, b[0], b[1], b[2], b[3]);
      uint64_t mine[4], got[4];
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        const uint64_t send = odd ? a[z] : b[z];  // what the partner's step needs
        mine[z] = odd ? b[z] : a[z];              // even: its high line, odd: its low line
        got[z] = __shfl_xor_sync(0xFFFFFFFFu, send, 1);
      }
      const uint64_t* hi_l = odd ? got : mine;
      const uint64_t* lo_l = odd ? mine : got;
      bh[u][0] = uint32_t(hi_l[0]), bh[u][1] = uint32_t(hi_l[0] >> 32), bh[u][2] = uint32_t(hi_l[1]);
      bh[u][3] = uint32_t(hi_l[1] >> 32), wh[u][0] = hi_l[2], wh[u][1] = hi_l[3];
      bl[u][0] = uint32_t(lo_l[0]), bl[u][1] = uint32_t(lo_l[0] >> 32), bl[u][2] = uint32_t(lo_l[1]);
      bl[u][3] = uint32_t(lo_l[1] >> 32), wl[u][0] = lo_l[2], wl[u][1] = lo_l[3];
      two[u] = true;  // the low line's data is always in bl / wl (the same line again when jl == jh)
    } else {
      load_line<W, true>(ix, jh, rh[u], bh[u], wh[u]);
      if (two[u]) load_line<W, true>(ix, jl, rl[u], bl[u], wl[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    if (!kBulk && !act[u]) continue;
    const uint32_t k = q[u].x, l = q[u].y;
    uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
    if (ok[u]) {
      occ4_from_line<W>(ix, bh[u], wh[u], l, rh[u], hi);
      if (k != 0u) {
        if (two[u])
          occ4_from_line<W>(ix, bl[u], wl[u], k - 1u, rl[u], lo);
        else
          occ4_from_line<W>(ix, bh[u], wh[u], k - 1u, rl[u], lo);
      }
    }
    const uint64_t i = first + uint64_t(u) * blockDim.x;
    if constexpr (kBulk) {
      uint4* sp = reinterpret_cast<uint4*>(stage + threadIdx.x * 8);
      sp[0] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      sp[1] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    } else {
      st_stream_256(out + i * 8, lo, hi);
    }
  }
  if constexpr (kBulk) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // these writes, then the async proxy's read
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t base = uint64_t(blockIdx.x) * blockDim.x;
      const uint32_t bytes = uint32_t(min(uint64_t(blockDim.x), count - base)) * 32u;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + base * 8),
                   "r"(uint32_t(__cvta_generic_to_shared(stage))), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the block's shared memory outlives the read
    }
  }
}

// Two lanes per Occ step (W = 2): lane 0 handles position k-1, lane 1
// position l, each loading ITS line in the same instruction.  When the two
// lines share a 128-byte chunk (64% of config-1 steps) the coalescer merges
// them into one L2 request, so requests per step drop from 1.75 (lines) to
// 1.36 (chunks); each lane counts one position and stores its 16 bytes.
// kBulk: the block's counts staged in shared memory and written by one bulk
// copy (see k_occ_pair).
template <bool kBulk = false>
__global__ void __launch_bounds__(256) k_occ_pair_2l(IndexView ix, const uint2* __restrict__ kl, uint64_t count,
                                                     uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  __shared__ __align__(128) uint32_t stage[kBulk ? 256 * 4 : 4];
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t i = t >> 1;
  const uint32_t role = uint32_t(t & 1u);  // 0: low (k-1), 1: high (l)
  if constexpr (kBulk) {
    const bool act = i < count;
    const uint2 q = act ? ld_stream_u2(kl + i) : make_uint2(1u, 0u);
    const uint32_t k = q.x, l = q.y;
    const bool ok = act && l <= ix.n && k <= l + 1u;
    if (act && !ok && role == 0u && err) atomicOr(err, 1u);
    const bool none = !ok || (role == 0u && k == 0u);
    const uint32_t p = role ? l : k - 1u;
    const uint32_t pp = none ? (ok ? l : 0u) : p;
    uint32_t b[4], r4[4] = {0u, 0u, 0u, 0u};
    uint64_t w[2];
    load_line<2, true>(ix, pp >> 6, pp & 63u, b, w);
    if (!none) occ4_from_line<2>(ix, b, w, p, p & 63u, r4);
    *reinterpret_cast<uint4*>(stage + threadIdx.x * 4) = make_uint4(r4[0], r4[1], r4[2], r4[3]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t base = uint64_t(blockIdx.x) * (blockDim.x >> 1);  // first pair of the block
      if (base < count) {
        const uint32_t bytes = uint32_t(min(uint64_t(blockDim.x >> 1), count - base)) * 32u;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + base * 8),
                     "r"(uint32_t(__cvta_generic_to_shared(stage))), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    return;
  }
  if (i >= count) return;
  const uint2 q = ld_stream_u2(kl + i);
  const uint32_t k = q.x, l = q.y;
  const bool ok = l <= ix.n && k <= l + 1u;
  if (!ok && role == 0u && err) atomicOr(err, 1u);
  const bool none = !ok || (role == 0u && k == 0u);  // Occ(., -1) = 0
  const uint32_t p = role ? l : k - 1u;
  const uint32_t pp = none ? (ok ? l : 0u) : p;  // a lane with nothing to count reads its partner's line
  uint32_t b[4], r4[4] = {0u, 0u, 0u, 0u};
  uint64_t w[2];
  load_line<2, true>(ix, pp >> 6, pp & 63u, b, w);
  if (!none) occ4_from_line<2>(ix, b, w, p, p & 63u, r4);
  uint4* dst = reinterpret_cast<uint4*>(out + i * 8 + role * 4);
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst), "r"(r4[0]),
               "r"(r4[1]), "r"(r4[2]), "r"(r4[3]), "l"(policy_evict_first())
               : "memory");
}

// Random-fetch microbenchmark (the ceiling of the HBM-resident Occ step):
// one random 32-byte read per thread from `bytes` of memory, addresses from a
// hash (tools/micro/gather*.cu measured 48 G/s on B200 for 4 GiB).
__global__ void k_random_fetch(const uint8_t* __restrict__ buf, uint64_t n_slots, uint64_t count, uint64_t seed,
                               unsigned long long* sink) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  const uint64_t slot = x % n_slots;
  uint64_t a0, a1, a2, a3;
  ld256<true>(buf + slot * 32, a0, a1, a2, a3);
  if ((a0 ^ a1 ^ a2 ^ a3) == 0x123456789ull) atomicAdd(sink, 1ull);
}

// Lane-cooperative Occ step for wide lines (W = 6: 2 lanes, W = 14: 4 lanes).
// The LANES lanes of a group each load one 32-byte sector of the same line in
// ONE instruction, so the line costs a single memory request (on B200 a
// random 64-byte request costs the same as a 32-byte one, 128 bytes 1.2x;
// tools/micro/gather3.cu), and count the fields of their own words; partial
// (T, hi, lo) popcounts are summed with xor-shuffles.  Fewer, denser lines
// mean fewer DRAM requests per step for HBM-resident indexes.
template <int W>
__device__ __forceinline__ void partial_counts(const uint64_t v[4], int sector, uint32_t r, uint32_t& t, uint32_t& h,
                                               uint32_t& l) {
  // sector 0 holds words 0, 1 (after the 16-byte checkpoint); sector j >= 1
  // holds words 4j-2 .. 4j+1
  const int k0 = sector == 0 ? 0 : 4 * sector - 2;
  const int nw = sector == 0 ? 2 : 4;
  t = h = l = 0;
#pragma unroll
  for (int q = 0; q < 4; q += 2) {
    if (q >= nw) break;
    const uint64_t wa = (sector == 0 ? v[2 + q] : v[q]), wb = (sector == 0 ? v[3 + q] : v[q + 1]);
    const uint64_t x0 = wa & word_mask(r, k0 + q), x1 = wb & word_mask(r, k0 + q + 1);
    const uint64_t lo = (x0 & kFieldLo) | ((x1 & kFieldLo) << 1);
    const uint64_t hi = ((x0 >> 1) & kFieldLo) | (x1 & ~kFieldLo);
    t += __popcll(lo & hi);
    h += __popcll(hi);
    l += __popcll(lo);
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_occ_pair_coop(IndexView ix, const uint2* __restrict__ kl, uint64_t count,
                                                       uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  constexpr int LANES = int(LineTraits<W>::kBytes / 32);
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const int sector = threadIdx.x % LANES;
  // the lanes of a group always agree on the pair index, so shuffles use the
  // group's own mask (groups of one warp may leave the loop at different times)
  const uint32_t gmask = ((1u << LANES) - 1u) << ((threadIdx.x & 31u) & ~uint32_t(LANES - 1));
  {
    const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LANES;  // one group per pair
    if (i >= count) return;  // the whole group leaves together
    const uint2 q = ld_stream_u2(kl + i);
    const uint32_t k = q.x, l = q.y;
    const bool ok = l <= ix.n && k <= l + 1u;
    if (!ok && sector == 0 && err) atomicOr(err, 1u);
    const uint32_t hh = ok ? l : 0u;
    const uint32_t ll = (ok && k != 0u) ? k - 1u : hh;
    const uint32_t jh = line_of<W>(hh), jl = line_of<W>(ll);
    const uint32_t rh = hh - jh * kC, rl = ll - jl * kC;
    uint64_t vh[4], vl[4];
    ld256<true>(ix.lines + size_t(jh) * LineTraits<W>::kBytes + 32 * sector, vh[0], vh[1], vh[2], vh[3]);
    const bool two = jl != jh;
    if (two) ld256<true>(ix.lines + size_t(jl) * LineTraits<W>::kBytes + 32 * sector, vl[0], vl[1], vl[2], vl[3]);
    uint32_t th, hh_, lh, tl, hl, ll_;
    partial_counts<W>(vh, sector, rh, th, hh_, lh);
    if (two)
      partial_counts<W>(vl, sector, rl, tl, hl, ll_);
    else
      partial_counts<W>(vh, sector, rl, tl, hl, ll_);
#pragma unroll
    for (int d = 1; d < LANES; d <<= 1) {
      th += __shfl_xor_sync(gmask, th, d);
      hh_ += __shfl_xor_sync(gmask, hh_, d);
      lh += __shfl_xor_sync(gmask, lh, d);
      tl += __shfl_xor_sync(gmask, tl, d);
      hl += __shfl_xor_sync(gmask, hl, d);
      ll_ += __shfl_xor_sync(gmask, ll_, d);
    }
    if (sector == 0) {
      uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
      if (ok) {
        const uint32_t bh[4] = {uint32_t(vh[0]), uint32_t(vh[0] >> 32), uint32_t(vh[1]), uint32_t(vh[1] >> 32)};
        hi[3] = bh[3] + th;
        hi[2] = bh[2] + hh_ - th;
        hi[1] = bh[1] + lh - th;
        hi[0] = bh[0] + rh + 1u - hh_ - lh + th - (l >= ix.sentinel_row ? 1u : 0u);
        if (k != 0u) {
          const uint64_t b01 = two ? vl[0] : vh[0], b23 = two ? vl[1] : vh[1];
          const uint32_t bl[4] = {uint32_t(b01), uint32_t(b01 >> 32), uint32_t(b23), uint32_t(b23 >> 32)};
          lo[3] = bl[3] + tl;
          lo[2] = bl[2] + hl - tl;
          lo[1] = bl[1] + ll_ - tl;
          lo[0] = bl[0] + rl + 1u - hl - ll_ + tl - (k - 1u >= ix.sentinel_row ? 1u : 0u);
        }
      }
      st_stream_256(out + i * 8, lo, hi);
    }
  }
}

}  // namespace fmg
