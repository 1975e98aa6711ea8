// B200-native FM-index engine: kernels and the C ABI of include/fmgpu.h.
//
// Kernels (all sm_100a, integer/popcount + random 32-byte gathers; no tensor
// cores — the Occ step has no GEMM shape):
//   k_build_lines   .fmi bucket records -> 32-byte lines          (index.py:24-36)
//   k_occ_pair      one thread per (k-1, l) pair, PER pairs/thread (occ.py:59-96)
//   k_exact         persistent, lane-refill backward search      (search.py:74-94)
//   k_inexact       persistent, lane-refill DFS with a per-thread
//                   stack and a lower-bound prune                (search.py:97-159)
//   k_psi / k_locate  predecessor walk to the sampled rows       (search.py:172-208)

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "fmgpu_internal.h"
#include "occ_device.cuh"

namespace fmg {

thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

#define FMG_CK(expr)                                                                      \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::fmg::CudaError(std::string(#expr) + " failed: " + cudaGetErrorString(e_)); \
  } while (0)

#define FMG_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) throw std::invalid_argument(msg); \
  } while (0)

// Restores the caller's current device on scope exit (the library must not
// disturb torch's or the application's device selection).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    FMG_CK(cudaGetDevice(&prev));
    if (prev != dev) FMG_CK(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Stream-ordered device allocation (pool-backed, cheap after warm-up).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t s) : stream(s) {
    if (count) FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&ptr), count * sizeof(T), s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), stream(o.stream) { o.ptr = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(stream, o.stream);
    return *this;
  }
  ~DevBuf() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------

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
template <int PER, int W>
__global__ void __launch_bounds__(256) k_occ_pair(IndexView ix, const uint2* __restrict__ kl, uint64_t count,
                                                  uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
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
    if (act[u] && !ok[u]) atomicOr(err, 1u);
    const uint32_t hh = ok[u] ? l : 0u;
    const uint32_t ll = (ok[u] && k != 0u) ? k - 1u : hh;
    const uint32_t jh = line_of<W>(hh), jl = line_of<W>(ll);
    rh[u] = hh - jh * kC;
    rl[u] = ll - jl * kC;
    two[u] = jl != jh;
    load_line<W, true>(ix, jh, rh[u], bh[u], wh[u]);
    if (two[u]) load_line<W, true>(ix, jl, rl[u], bl[u], wl[u]);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    if (!act[u]) continue;
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
    st_stream_256(out + i * 8, lo, hi);
  }
}

// Two lanes per Occ step (W = 2): lane 0 handles position k-1, lane 1
// position l, each loading ITS line in the same instruction.  When the two
// lines share a 128-byte chunk (64% of config-1 steps) the coalescer merges
// them into one L2 request, so requests per step drop from 1.75 (lines) to
// 1.36 (chunks); each lane counts one position and stores its 16 bytes.
__global__ void __launch_bounds__(256) k_occ_pair_2l(IndexView ix, const uint2* __restrict__ kl, uint64_t count,
                                                     uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t i = t >> 1;
  const uint32_t role = uint32_t(t & 1u);  // 0: low (k-1), 1: high (l)
  if (i >= count) return;
  const uint2 q = ld_stream_u2(kl + i);
  const uint32_t k = q.x, l = q.y;
  const bool ok = l <= ix.n && k <= l + 1u;
  if (!ok && role == 0u) atomicOr(err, 1u);
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
    if (!ok && sector == 0) atomicOr(err, 1u);
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

// Pattern sources for the search kernels.
struct PackedPatterns {  // fixed length m <= 32, char j in bits 2j..2j+1
  const uint64_t* words;
  uint32_t m;
  __device__ __forceinline__ uint32_t length(uint64_t) const { return m; }
};
struct CodePatterns {  // codes[offsets[q] .. offsets[q+1])
  const uint8_t* codes;
  const uint64_t* offsets;
  const ulonglong2* packed = nullptr;  // inexact, m <= 64: 2-bit packed copy (k_pack_patterns)
  const uint64_t* packed1 = nullptr;   // inexact, fixed m <= 32 given packed by the caller
  uint32_t fixed_m = 0;
  const uint64_t* dbits = nullptr;     // inexact, m <= 64: lower-bound segment ends (k_dbound)
};

// Exact backward search, one pattern per thread at a time.  When a lane's
// pattern finishes (matched or emptied — the reference stops at the FIRST
// empty interval, search.py:91-92) the lane immediately takes the next
// pattern of its grid-stride sequence, so warps stay full while per-pattern
// step counts vary from 1 to m-1.
template <bool kPacked, int W>
__global__ void __launch_bounds__(256) k_exact(IndexView ix, PackedPatterns pp, CodePatterns cp, uint64_t count,
                                               uint2* __restrict__ out, unsigned long long* __restrict__ steps) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t my_steps = 0;
  uint64_t pat = 0;          // packed form
  const uint8_t* codes = nullptr;  // general form
  int i = -1;
  uint32_t k = 1, l = 0;
  auto start = [&](uint64_t qq) {
    uint32_t m, b;
    if (kPacked) {
      pat = pp.words[qq];
      m = pp.m;
      b = uint32_t(pat >> (2 * (m - 1))) & 3u;
    } else {
      const uint64_t o0 = cp.offsets[qq], o1 = cp.offsets[qq + 1];
      codes = cp.codes + o0;
      m = uint32_t(o1 - o0);
      b = codes[m - 1];
    }
    k = c_of(ix, b) + 1u;  // init_interval, search.py:50-57
    l = c_of(ix, b + 1u);
    i = int(m) - 2;
  };
  if (q >= count) return;
  start(q);
  while (true) {
    if (i < 0 || k > l) {
      out[q] = make_uint2(k, l);
      q += stride;
      if (q >= count) break;
      start(q);
      continue;
    }
    const uint32_t sym = kPacked ? (uint32_t(pat >> (2 * i)) & 3u) : uint32_t(__ldg(codes + i));
    --i;
    // extend_backward, search.py:60-71: k' = c[b] + Occ(b, k-1) + 1, l' = c[b] + Occ(b, l)
    constexpr uint32_t kC = LineTraits<W>::kChars;
    uint32_t bh[4], bl[4];
    uint64_t wh[W], wl[W];
    const uint32_t low = k - 1u;  // k >= 1 on every non-empty interval here
    const uint32_t jh = line_of<W>(l), jl = line_of<W>(low);
    const uint32_t rh = l - jh * kC, rl = low - jl * kC;
    load_line<W, false>(ix, jh, rh, bh, wh);
    uint32_t ol;
    if (jl != jh) {
      load_line<W, false>(ix, jl, rl, bl, wl);
      ol = occ1_from_line<W>(ix, bl, wl, low, rl, sym);
    } else {
      ol = occ1_from_line<W>(ix, bh, wh, low, rl, sym);
    }
    const uint32_t oh = occ1_from_line<W>(ix, bh, wh, l, rh, sym);
    const uint32_t cs = c_of(ix, sym);
    k = cs + ol + 1u;
    l = cs + oh;
    ++my_steps;
  }
  if (steps) atomicAdd(steps, (unsigned long long)my_steps);
}

// ----- bounded-difference search -----------------------------------------

// Lower-bound pass of the inexact search as its own kernel (patterns of
// length <= 64): one thread per pattern extends right to left with resets;
// every time W[pos..seg_end] is absent from the text, bit seg_end is set and
// the search restarts from the root at pos-1.  D(i) = popcount of the bits
// <= i (see k_inexact).  Running it apart keeps the DFS kernel's lanes in
// one phase.
template <int W>
__global__ void __launch_bounds__(256) k_dbound(IndexView ix, CodePatterns cp, uint64_t count,
                                                uint64_t* __restrict__ dbits_out, unsigned long long* steps) {
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
  uint64_t bits = 0;
  uint32_t k = 0, l = ix.n;
  int seg_end = m - 1;
  uint32_t my_steps = 0;
  for (int pos = m - 1; pos >= 0; --pos) {
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
      ++my_steps;
    }
    if (k2 > l2) {  // W[pos..seg_end] is absent from the text
      bits |= 1ull << seg_end;
      k = 0;
      l = ix.n;
      seg_end = pos - 1;
    } else {
      k = k2;
      l = l2;
    }
  }
  dbits_out[q] = bits;
  if (steps) atomicAdd(steps, (unsigned long long)my_steps);
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
template <bool kShort, int W>
__global__ void __launch_bounds__(128) k_inexact(IndexView ix, CodePatterns cp, const uint32_t* __restrict__ list,
                                                 uint64_t count, uint32_t z, InexactScratch sc, InexactOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t S = sc.S, nt = blockDim.x, tid = threadIdx.x;
  uint2* s_kl = reinterpret_cast<uint2*>(smem);               // [S][nt]
  uint32_t* s_ib = reinterpret_cast<uint32_t*>(s_kl + S * nt);  // [S][nt]
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= sc.T) return;
  uint64_t my_steps = 0;
  const uint64_t wbase = t >> 5, lane = t & 31u;
  auto HI = [&](uint32_t e) -> uint64_t { return (wbase * (2u * sc.R) + e) * 32u + lane; };
  auto LI = [&](uint32_t e) -> uint64_t { return (wbase * sc.R + e) * 32u + lane; };
  uint32_t epoch = 0;  // per-thread pattern counter: table slots of older patterns read as empty
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
  uint32_t cb = 0, ck = 0, cl = 0;

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
          ck = 0u;
          cl = ix.n;
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
          cb = ib & 0xFFFFu;
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

    // ---- one Occ step: the eight values at (k-1, l) ----
    uint32_t lo[4], hi[4];
    occ_step<W, false>(ix, k, l, lo, hi);
    ++my_steps;

    if (phase == 0) {
      const uint32_t b = sym_at(pos);
      const uint32_t cbase = c_of(ix, b);
      const uint32_t k2 = cbase + sel4(lo, b) + 1u, l2 = cbase + sel4(hi, b);
      if (k2 > l2) {  // W[pos..seg_end] is absent from the text
        if (kShort)
          dbits |= 1ull << seg_end;
        else
          sc.dlb[DI(uint32_t(seg_end))] = 1;
        kd = 0;
        ld = ix.n;
        seg_end = pos - 1;
      } else {
        kd = k2;
        ld = l2;
      }
      --pos;
      continue;
    }

    // ---- DFS expansion of the register node (search.py:135-152) ----
    const int i = ci;
    const uint32_t budget = cb;
    const uint32_t want = sym_at(i);
    const uint32_t cw = c_of(ix, want);
    const uint32_t kw = cw + sel4(lo, want) + 1u, lw = cw + sel4(hi, want);
    if (budget == 0) {
      // budget-0 node: only the match child, continued in registers
      if (kw > lw) {
        cur_valid = false;
      } else if (i == 0) {
        record(kw, lw, z);
        cur_valid = false;
      } else {
        ci = i - 1;
        ck = kw;
        cl = lw;
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
    uint32_t k2[4], l2[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      k2[b] = ix.c[b] + lo[b] + 1u;
      l2[b] = ix.c[b] + hi[b];
    }
    if (at0) {  // children with i - 1 < 0 are results (rare)
      if (kw <= lw) record(kw, lw, z - budget);
      record(k, l, z - bm1);  // skip
#pragma unroll
      for (uint32_t b = 0; b < 4; ++b)
        if (b != want && k2[b] <= l2[b]) record(k2[b], l2[b], z - bm1);  // mismatch
    }
    auto push_if = [&](bool cond, int pi, uint32_t pb, uint32_t pk, uint32_t pl) {
      if (cond) {
        if (sp == S) {
          overflow = true;
        } else {
          s_kl[sp * nt + tid] = make_uint2(pk, pl);
          s_ib[sp * nt + tid] = (uint32_t(pi + 1) << 16) | pb;
          ++sp;
        }
      }
    };
    push_if(ok_match && kw <= lw, i - 1, budget, kw, lw);  // match
    push_if(ok_prev, i - 1, bm1, k, l);                      // skip
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b) {
      const bool ne = k2[b] <= l2[b];
      push_if(ok_cur && ne, i, bm1, k2[b], l2[b]);                 // insert
      push_if(ok_prev && ne && b != want, i - 1, bm1, k2[b], l2[b]);  // mismatch
    }
    cur_valid = false;  // the next iteration pops the top (the last child pushed)
  }
  if (out.steps) atomicAdd(out.steps, (unsigned long long)my_steps);
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
  uint32_t my_steps = 0;
  int i = m - 1;
  uint32_t k = 0, l = ix.n;
  bool alive = z1_dlb(dbits, m - 1) <= 1u;  // root (m-1, 1, 0, n), search.py:125
  while (alive) {
    uint32_t lo[4], hi[4];
    occ_step<W, false>(ix, k, l, lo, hi);
    ++my_steps;
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
      if (k2[want & 3u] <= l2[want & 3u]) ++rc;  // match with budget kept
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
      if (k2[want & 3u] <= l2[want & 3u]) rput(k2[want & 3u], l2[want & 3u], 0u);
      break;
    }
    // continue along the match child (i-1, 1)
    const uint32_t kw = sel4(k2, want), lw = sel4(l2, want);
    if (kw > lw || z1_dlb(dbits, i - 1) > 1u) break;
    k = kw;
    l = lw;
    --i;
  }
  if (steps) atomicAdd(steps, (unsigned long long)my_steps);
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
  uint32_t my_steps = 0;
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
      ++my_steps;
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
  if (steps) atomicAdd(steps, (unsigned long long)my_steps);
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
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint64_t a = offsets[q], b = offsets[q + 1];
  if (q == 0 && a != 0) atomicOr(err, 4u);
  if (b <= a) {
    atomicOr(err, 1u);
    return;
  }
  atomicMax(max_len, (unsigned long long)(b - a));
  for (uint64_t j = a; j < b; ++j)
    if (codes[j] > 3) atomicOr(err, 2u);
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

__global__ void k_widen_counts(uint64_t count, const uint32_t* __restrict__ c32, uint64_t* __restrict__ c64) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < count) c64[q] = c32[q];
}

// ----- position recovery ---------------------------------------------------

// psi_inverse_fused (search.py:172-186): symbol at row i and its
// predecessor row c[sym] + Occ(sym, i), in one line access.
template <int W>
__device__ __forceinline__ uint32_t psi_step(const IndexView& ix, uint32_t row, uint32_t& sym) {
  uint32_t b[4];
  uint64_t w[W];
  const uint32_t j = line_of<W>(row), r = row - j * LineTraits<W>::kChars;
  load_line<W, false>(ix, j, r, b, w);
  sym = field_at<W>(w, r);
  return c_of(ix, sym) + occ1_from_line<W>(ix, b, w, row, r, sym);
}

template <int W>
__global__ void k_psi(IndexView ix, const uint32_t* __restrict__ rows, uint64_t count, uint8_t* __restrict__ out_sym,
                      uint32_t* __restrict__ out_row, uint32_t* __restrict__ err) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint32_t row = rows[q];
  if (row > ix.n) {
    atomicOr(err, 1u);
    out_sym[q] = 255;
    out_row[q] = 0xFFFFFFFFu;
    return;
  }
  if (row == ix.sentinel_row) {
    out_sym[q] = 255;
    out_row[q] = 0xFFFFFFFFu;
    return;
  }
  uint32_t sym;
  const uint32_t prev = psi_step<W>(ix, row, sym);
  out_sym[q] = uint8_t(sym);
  out_row[q] = prev;
}

// locate_row (search.py:189-208): walk predecessors until the row is sampled
// (row % 32 == 0 — samples are taken by ROW, index.py:93, so the walk length
// is geometric-like with mean ~32, not bounded by 32) or is the sentinel row.
// Grid-stride lane refill keeps warps full despite the varying walk lengths.
template <int W>
__global__ void __launch_bounds__(256) k_locate(IndexView ix, const uint32_t* __restrict__ rows, uint64_t count,
                                                uint32_t* __restrict__ out_pos, uint32_t* __restrict__ err) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < count; q += stride) {
    uint32_t row = rows[q];
    if (row > ix.n) {
      atomicOr(err, 1u);
      out_pos[q] = 0xFFFFFFFFu;
      continue;
    }
    uint32_t steps = 0;
    while (true) {
      if (row == ix.sentinel_row) {
        out_pos[q] = steps;
        break;
      }
      if ((row & 31u) == 0u) {
        out_pos[q] = ix.samples[row >> 5] + steps;
        break;
      }
      uint32_t sym;
      row = psi_step<W>(ix, row, sym);
      ++steps;
      if (steps > ix.n + 1u) {  // corrupt index (search.py:207-208)
        atomicOr(err, 2u);
        out_pos[q] = 0xFFFFFFFFu;
        break;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------

int sm_count(int device) {
  int v = 0;
  FMG_CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

}  // namespace fmg

struct fmg_index {
  int device = 0;
  uint64_t n = 0, sentinel_row = 0, c[5] = {0, 0, 0, 0, 0};
  uint64_t n_buckets = 0, n_lines = 0, n_samples = 0;
  int words = 2;  // line layout: W words of 32 chars per line (occ_device.cuh)
  uint8_t* lines = nullptr;
  uint32_t* samples = nullptr;
  uint32_t* err = nullptr;  // sticky device-side input error flags
  int sms = 148;

  fmg::IndexView view() const {
    fmg::IndexView v;
    v.lines = lines;
    v.samples = samples;
    v.n = uint32_t(n);
    v.sentinel_row = uint32_t(sentinel_row);
    for (int s = 0; s < 5; ++s) v.c[s] = uint32_t(c[s]);
    return v;
  }
};

struct fmg_matches {
  int device = 0;
  uint64_t patterns = 0, total = 0, steps = 0;
  uint64_t* row_off = nullptr;  // device, patterns + 1
  uint32_t* k = nullptr;        // device, total
  uint32_t* l = nullptr;
  uint8_t* diffs = nullptr;
};

namespace {

using namespace fmg;

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Line layout.  W = 2 (32-byte lines, one sector per Occ) is the default for
// every index size: measured on B200, a random L2 miss costs one DRAM request
// (~48 G requests/s chip-wide) whatever its size up to 64 B, and W = 6 / 14
// lines read by one thread need 2-4 requests and 3-7x the popcount work
// (tools/size_sweep.py, profiles/).  FMG_LINE_WORDS=2|6|14 overrides (the
// tests exercise every layout).
int choose_words(uint64_t n_buckets) {
  if (const char* env = std::getenv("FMG_LINE_WORDS")) {
    const int w = std::atoi(env);
    FMG_REQUIRE(w == 2 || w == 6 || w == 14, "FMG_LINE_WORDS must be 2, 6 or 14");
    return w;
  }
  (void)n_buckets;
  return 2;
}

void check_index(const fmg_index* ix) { FMG_REQUIRE(ix != nullptr, "null index handle"); }

// Reads and clears the sticky input-error flags (synchronises `stream`).
void take_input_error(const fmg_index* ix, cudaStream_t stream, const char* what) {
  uint32_t h = 0;
  FMG_CK(cudaMemcpyAsync(&h, ix->err, sizeof(h), cudaMemcpyDeviceToHost, stream));
  FMG_CK(cudaStreamSynchronize(stream));
  if (h) {
    FMG_CK(cudaMemsetAsync(ix->err, 0, sizeof(uint32_t), stream));
    FMG_CK(cudaStreamSynchronize(stream));
    if (h & 2u) throw std::runtime_error("predecessor walk did not terminate; index is corrupt");
    throw std::invalid_argument(what);
  }
}

// Runs f(std::integral_constant<int, W>) for the index's line layout.
template <typename F>
void with_words(const fmg_index* ix, F&& f) {
  switch (ix->words) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 14: f(std::integral_constant<int, 14>{}); break;
    default: throw std::invalid_argument("unsupported line layout");
  }
}

constexpr int kOccPer = 1;

template <int PER>
void launch_occ_pair_t(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, cudaStream_t s,
                       int threads) {
  const uint64_t per_block = uint64_t(threads) * PER;
  const uint64_t blocks = (count + per_block - 1) / per_block;
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    // two lanes per step only for HBM-resident line arrays (> 64 MB): +4% on
    // config 1-H, -8% on the L2-resident config 1 (profiles/r01_occ.md)
    const char* e2l = std::getenv("FMG_OCC_2LANE");  // A/B hook
    const bool two_lane = e2l ? std::atoi(e2l) != 0 : ix->n_lines * 32ull > (64ull << 20);
    if (W == 2 && two_lane) {
      k_occ_pair_2l<<<dim3(unsigned((2 * count + 255) / 256)), 256, 0, s>>>(
          ix->view(), reinterpret_cast<const uint2*>(kl), count, out, ix->err);
    } else if (W == 2) {
      k_occ_pair<PER, W><<<dim3(unsigned(blocks)), threads, 0, s>>>(ix->view(), reinterpret_cast<const uint2*>(kl),
                                                                      count, out, ix->err);
    } else {  // wide lines: lane-cooperative, persistent grid-stride
      constexpr int LANES = int(LineTraits<W>::kBytes / 32);
      const uint64_t nb = (count * LANES + 255) / 256;
      k_occ_pair_coop<W><<<dim3(unsigned(std::max<uint64_t>(nb, 1))), 256, 0, s>>>(
          ix->view(), reinterpret_cast<const uint2*>(kl), count, out, ix->err);
    }
  });
  FMG_CK(cudaGetLastError());
}

void launch_occ_pair(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, cudaStream_t s,
                     int per = kOccPer, int threads = 128) {
  if (count == 0) return;
  FMG_REQUIRE(threads == 128 || threads == 256, "threads must be 128 or 256");
  switch (per) {
    case 1: launch_occ_pair_t<1>(ix, kl, count, out, s, threads); break;
    case 2: launch_occ_pair_t<2>(ix, kl, count, out, s, threads); break;
    case 4: launch_occ_pair_t<4>(ix, kl, count, out, s, threads); break;
    default: throw std::invalid_argument("per must be 1, 2 or 4");
  }
}

unsigned persistent_blocks(const fmg_index* ix, const void* kernel, int threads, uint64_t work) {
  int per_sm = 0;
  FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
  static const int mult = [] {
    const char* e = std::getenv("FMG_GRID_MULT");  // tuning hook: waves of the persistent grid
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  uint64_t blocks = uint64_t(std::max(per_sm, 1)) * ix->sms * mult;
  const uint64_t need = (work + threads - 1) / threads;
  return unsigned(std::max<uint64_t>(1, std::min(blocks, need)));
}

// Grid for the lane-refill search kernels: about kPerThread queries per
// thread, i.e. many more blocks than fit at once.  Measured on B200 (config
// 4, tools/prof_exact.py): letting the block scheduler refill SMs beats a
// persistent one-wave grid whose lanes refill themselves (2.56 -> 3.3 G
// seeds/s), because a self-refilling lane stalls the rest of its warp.
unsigned wave_blocks(const fmg_index* ix, const void* kernel, int threads, uint64_t work) {
  constexpr uint64_t kPerThread = 4;
  const uint64_t resident = persistent_blocks(ix, kernel, threads, work);
  const uint64_t waves = (work + threads * kPerThread - 1) / (threads * kPerThread);
  return unsigned(std::min<uint64_t>(std::max<uint64_t>(resident, waves), 1u << 30));
}

void launch_exact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, uint32_t* kl_out,
                         cudaStream_t s, unsigned long long* steps) {
  if (count == 0) return;
  PackedPatterns pp{packed, m};
  CodePatterns cp{nullptr, nullptr};
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)k_exact<true, W>, 256, count);
    k_exact<true, W><<<blocks, 256, 0, s>>>(ix->view(), pp, cp, count, reinterpret_cast<uint2*>(kl_out), steps);
  });
  FMG_CK(cudaGetLastError());
}

void launch_exact_codes(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                        uint32_t* kl_out, cudaStream_t s, unsigned long long* steps) {
  if (count == 0) return;
  PackedPatterns pp{nullptr, 0};
  CodePatterns cp{codes, offsets};
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)k_exact<false, W>, 256, count);
    k_exact<false, W><<<blocks, 256, 0, s>>>(ix->view(), pp, cp, count, reinterpret_cast<uint2*>(kl_out), steps);
  });
  FMG_CK(cudaGetLastError());
}

void launch_locate(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos, cudaStream_t s) {
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)fmg::k_locate<W>, 256, count);
    fmg::k_locate<W><<<blocks, 256, 0, s>>>(ix->view(), rows, count, out_pos, ix->err);
  });
  FMG_CK(cudaGetLastError());
}

// Validates a device pattern batch (k_check_patterns) and returns the
// longest pattern; throws invalid_argument like the reference's ValueErrors.
uint64_t validate_patterns_device(const uint8_t* codes, const uint64_t* offsets, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  DevBuf<unsigned long long> ml(1, s);
  DevBuf<uint32_t> err(1, s);
  FMG_CK(cudaMemsetAsync(ml.ptr, 0, 8, s));
  FMG_CK(cudaMemsetAsync(err.ptr, 0, 4, s));
  k_check_patterns<<<unsigned((count + 255) / 256), 256, 0, s>>>(codes, offsets, count, ml.ptr, err.ptr);
  FMG_CK(cudaGetLastError());
  unsigned long long h_ml = 0;
  uint32_t h_err = 0;
  FMG_CK(cudaMemcpyAsync(&h_ml, ml.ptr, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaMemcpyAsync(&h_err, err.ptr, 4, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  FMG_REQUIRE(!(h_err & 4u), "pattern offsets must start at 0");
  FMG_REQUIRE(!(h_err & 1u), "pattern is empty");
  FMG_REQUIRE(!(h_err & 2u), "symbol code outside [0, 4)");
  return h_ml;
}


// z = 1 through k_spine / k_chain; false when a queue overflowed (the caller
// then runs the DFS engine, which has no such limit).  Fills res on success.
bool run_z1(const fmg_index* ix, const CodePatterns& cp, uint64_t count, uint64_t m, cudaStream_t s,
            unsigned long long* steps, fmg_matches* res) {
  static const bool trace = std::getenv("FMG_TRACE") != nullptr;
  cudaEvent_t ev[4] = {};
  if (trace)
    for (auto& e : ev) cudaEventCreate(&e);
  if (trace) cudaEventRecord(ev[0], s);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = size_t(8) << 30;
  // worst case 8 continuations per spine node and m + 1 spine nodes; in
  // practice far fewer, so cap by memory and detect overflow
  const uint64_t worst = count * 8 * (m + 1);
  const uint64_t budget_entries = std::max<uint64_t>(1u << 20, free_b / 4 / sizeof(Z1Node));
  const uint64_t node_cap = std::min<uint64_t>(worst, budget_entries);
  const uint64_t raw_cap = std::min<uint64_t>(worst + count, budget_entries / 2);
  DevBuf<Z1Node> nodes(node_cap, s);
  DevBuf<Z1Raw> raws(raw_cap, s);
  DevBuf<unsigned long long> ctr(2, s);
  FMG_CK(cudaMemsetAsync(ctr.ptr, 0, 16, s));
  Z1Queues qu{nodes.ptr, ctr.ptr, node_cap, raws.ptr, ctr.ptr + 1, raw_cap};
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    k_spine<W><<<unsigned((count + 255) / 256), 256, 0, s>>>(ix->view(), cp, count, qu, steps);
  });
  FMG_CK(cudaGetLastError());
  unsigned long long n_nodes = 0;
  FMG_CK(cudaMemcpyAsync(&n_nodes, ctr.ptr, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  if (n_nodes > node_cap) return false;
  if (trace) cudaEventRecord(ev[1], s);
  if (n_nodes) {
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      const unsigned nb = persistent_blocks(ix, (const void*)k_chain<W>, 256, n_nodes);
      k_chain<W><<<nb, 256, 0, s>>>(ix->view(), cp, nodes.ptr, n_nodes, qu, steps);
    });
    FMG_CK(cudaGetLastError());
  }
  unsigned long long n_raw = 0;
  FMG_CK(cudaMemcpyAsync(&n_raw, ctr.ptr + 1, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  if (n_raw > raw_cap) return false;
  if (trace) cudaEventRecord(ev[2], s);
  // group raw results by pattern (counting sort), sort each segment by (k, l)
  DevBuf<uint32_t> per_q(count, s);
  DevBuf<uint64_t> seg(count + 1, s), cursor(count, s), c64(count, s);
  FMG_CK(cudaMemsetAsync(per_q.ptr, 0, count * 4, s));
  FMG_CK(cudaMemsetAsync(seg.ptr, 0, 8, s));
  if (n_raw) k_z1_hist<<<unsigned((n_raw + 255) / 256), 256, 0, s>>>(raws.ptr, n_raw, per_q.ptr);
  k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  size_t tb = 0;
  FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, c64.ptr, seg.ptr + 1, count, s));
  DevBuf<uint8_t> tmp(tb, s);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, seg.ptr + 1, count, s));
  FMG_CK(cudaMemcpyAsync(cursor.ptr, seg.ptr, count * 8, cudaMemcpyDeviceToDevice, s));
  const uint64_t nr = std::max<uint64_t>(n_raw, 1);
  DevBuf<uint64_t> keys(nr, s), keys2(nr, s);
  DevBuf<uint8_t> used(nr, s), used2(nr, s);
  if (n_raw) {
    k_z1_scatter<<<unsigned((n_raw + 255) / 256), 256, 0, s>>>(raws.ptr, n_raw, cursor.ptr, keys.ptr, used.ptr);
    FMG_REQUIRE(n_raw < (1ull << 31), "too many inexact results for one call");
    size_t sb = 0;
    FMG_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, keys.ptr, keys2.ptr, used.ptr, used2.ptr, int(n_raw),
                                               int(count), seg.ptr, seg.ptr + 1, s));
    DevBuf<uint8_t> stmp(sb, s);
    FMG_CK(cub::DeviceSegmentedSort::SortPairs(stmp.ptr, sb, keys.ptr, keys2.ptr, used.ptr, used2.ptr, int(n_raw),
                                               int(count), seg.ptr, seg.ptr + 1, s));
  }
  k_z1_unique_count<<<unsigned((count + 255) / 256), 256, 0, s>>>(keys2.ptr, used2.ptr, seg.ptr, count, per_q.ptr);
  k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, res->row_off + 1, count, s));
  uint64_t total = 0;
  FMG_CK(cudaMemcpyAsync(&total, res->row_off + count, 8, cudaMemcpyDeviceToHost, s));
  unsigned long long st = 0;
  FMG_CK(cudaMemcpyAsync(&st, steps, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  res->total = total;
  res->steps = st;
  FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->k), std::max<uint64_t>(total, 1) * 4, s));
  FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->l), std::max<uint64_t>(total, 1) * 4, s));
  FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->diffs), std::max<uint64_t>(total, 1), s));
  k_z1_unique_write<<<unsigned((count + 255) / 256), 256, 0, s>>>(keys2.ptr, used2.ptr, seg.ptr, res->row_off,
                                                                  count, res->k, res->l, res->diffs);
  FMG_CK(cudaGetLastError());
  if (trace) cudaEventRecord(ev[3], s);
  FMG_CK(cudaStreamSynchronize(s));
  if (trace) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    fprintf(stderr, "[fmg] z1 engine: %llu patterns, spine+queue %.3f ms (%llu continuations), chains %.3f ms, "
            "dedup/sort %.3f ms (%llu raw -> %llu results)\n", (unsigned long long)count, a, n_nodes, b, c,
            n_raw, (unsigned long long)total);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  return true;
}

fmg_matches* run_inexact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                         uint64_t max_len, int max_diff, cudaStream_t s, const uint64_t* packed1 = nullptr) {
  FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
  FMG_REQUIRE(max_diff <= 0xFFFF, "difference budget above 65535 is not supported");
  FMG_REQUIRE(max_len < 0xFFFF, "pattern longer than 65534 is not supported");
  FMG_REQUIRE(count < 0xFFFFFFFFull, "too many patterns in one call");
  auto* res = new fmg_matches();
  res->device = ix->device;
  res->patterns = count;
  try {
    FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->row_off), (count + 1) * sizeof(uint64_t), s));
    FMG_CK(cudaMemsetAsync(res->row_off, 0, sizeof(uint64_t), s));
    if (count == 0) {
      FMG_CK(cudaStreamSynchronize(s));
      return res;
    }
    const uint32_t z = uint32_t(max_diff);
    const bool short_pat = max_len <= 64;
    const void* kfn = nullptr;
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      kfn = short_pat ? (const void*)k_inexact<true, W> : (const void*)k_inexact<false, W>;
    });
    int smem_optin = 0;
    FMG_CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix->device));

    DevBuf<uint64_t> res_off(count, s);
    DevBuf<uint32_t> res_cnt(count, s);
    DevBuf<uint8_t> res_pass(count, s);
    DevBuf<unsigned long long> counters(5, s);  // total, fail_count, steps, queue cursor, unsorted
    DevBuf<uint32_t> unsorted_list(count, s);
    DevBuf<uint32_t> too_big(1, s);
    FMG_CK(cudaMemsetAsync(too_big.ptr, 0, 4, s));
    bool need_cub_sort = false;
    FMG_CK(cudaMemsetAsync(res_pass.ptr, 0xFF, count, s));
    FMG_CK(cudaMemsetAsync(counters.ptr + 2, 0, sizeof(unsigned long long), s));
    FMG_CK(cudaMemsetAsync(counters.ptr + 4, 0, sizeof(unsigned long long), s));

    DevBuf<ulonglong2> packed((short_pat && !packed1) ? count : 0, s);
    if (short_pat && !packed1) {
      k_pack_patterns<<<unsigned((count + 255) / 256), 256, 0, s>>>(codes, offsets, count, packed.ptr);
      FMG_CK(cudaGetLastError());
    }
    DevBuf<uint64_t> dbits(short_pat ? count : 0, s);
    if (short_pat) {
      CodePatterns cpd{codes, offsets, packed.ptr, packed1, uint32_t(max_len)};
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        k_dbound<W><<<unsigned((count + 255) / 256), 256, 0, s>>>(ix->view(), cpd, count, dbits.ptr,
                                                                    counters.ptr + 2);
      });
      FMG_CK(cudaGetLastError());
    }
    // z = 1 on an L2-resident index: the level-synchronous engine (uniform
    // warps).  On HBM-resident indexes the DFS engine wins: its chains start
    // from intervals already in L1/L2, while queued continuations re-fetch
    // pattern, bound and first line from DRAM (tools/prof_c3.py).
    const bool force_dfs = std::getenv("FMG_INEXACT_DFS") != nullptr;  // read per call (tests flip it)
    uint64_t line_bytes = 0;
    with_words(ix, [&](auto wt) { line_bytes = ix->n_lines * fmg::LineTraits<decltype(wt)::value>::kBytes; });
    if (z == 1 && short_pat && !force_dfs && line_bytes <= (uint64_t(64) << 20)) {
      CodePatterns cpz{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      if (run_z1(ix, cpz, count, max_len, s, counters.ptr + 2, res)) return res;
      // queues overflowed: fall through to the DFS engine (same results)
    }
    std::vector<DevBuf<uint2>> pass_kl;
    std::vector<DevBuf<uint8_t>> pass_d;
    DevBuf<uint32_t> lists[2] = {DevBuf<uint32_t>(count, s), DevBuf<uint32_t>(count, s)};
    const uint32_t* list = nullptr;  // pass 0: every pattern
    uint64_t pending = count;
    // R: results per pattern before a retry (per-thread hash table of 2R
    // slots).  cap: results per pass (9 bytes each) before patterns finishing
    // later are retried — sized from free memory so a pass rarely fills it.
    uint32_t R = 256;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = size_t(8) << 30;
    uint64_t cap = std::max<uint64_t>(count * 16, 1u << 20);
    cap = std::min<uint64_t>(cap, std::max<uint64_t>(1u << 20, free_b / 4 / 9));
    // Stack: depth <= 8(z+1) with the budget-ordered pushes of k_inexact;
    // 9(m+z+1)+2 bounds any visiting order.  Grown on overflow.
    const uint32_t S_max = uint32_t(9 * (max_len + z + 1) + 2);
    // The stack is budget-monotone: at most one budget-z entry (the pending
    // spine child) and at most 9 entries per lower budget level, so 9z + 2
    // slots suffice.  Kept small on purpose: shared memory and L1 share the
    // SM's SRAM, and for HBM-resident indexes the L1 left over is worth 30%
    // (config 3: S = 20 -> 667 ms, S = 10 -> 447 ms per 14M seeds).
    uint32_t S = std::min<uint32_t>(S_max, 9 * z + 2);
    if (const char* e = std::getenv("FMG_STACK_S")) S = std::max<uint32_t>(2, uint32_t(std::atoi(e)));  // A/B
    for (int pass = 0; pending > 0; ++pass) {
      FMG_REQUIRE(pass < 250, "inexact search did not converge");
      int nt = 128;
      while (nt > 32 && size_t(S) * 12 * nt > size_t(96) << 10) nt /= 2;
      const size_t smem = size_t(S) * 12 * nt;
      FMG_REQUIRE(smem <= size_t(smem_optin), "inexact search stack does not fit in shared memory");
      FMG_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int per_sm = 0;
      FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, nt, smem));
      per_sm = std::max(per_sm, 1);
      // threads: full residency, bounded by a scratch budget of ~2 GiB
      const uint64_t per_thread = uint64_t(R) * (2 * 16 + 4) + (short_pat ? 0 : max_len);
      uint64_t T = uint64_t(per_sm) * ix->sms * nt;
      T = std::min<uint64_t>(T, std::max<uint64_t>(nt, std::max<uint64_t>(2ull << 30, free_b / 8) / per_thread));
      T = std::min<uint64_t>(T, ((pending + nt - 1) / nt) * nt);
      T = std::max<uint64_t>(nt, (T / nt) * nt);
      InexactScratch sc{};
      DevBuf<uint4> table(uint64_t(2 * R) * T, s);
      DevBuf<uint32_t> slots(uint64_t(R) * T, s);
      DevBuf<uint8_t> dl(short_pat ? 0 : max_len * T, s);
      FMG_CK(cudaMemsetAsync(table.ptr, 0, uint64_t(2 * R) * T * sizeof(uint4), s));  // epoch 0 = empty
      sc.table = table.ptr;
      sc.slots = slots.ptr;
      sc.dlb = dl.ptr;
      sc.S = S;
      sc.R = R;
      sc.Mmax = uint32_t(max_len);
      sc.T = T;
      pass_kl.emplace_back(cap, s);
      pass_d.emplace_back(cap, s);
      FMG_CK(cudaMemsetAsync(counters.ptr, 0, 2 * sizeof(unsigned long long), s));
      FMG_CK(cudaMemsetAsync(counters.ptr + 3, 0, sizeof(unsigned long long), s));
      InexactOut o{};
      o.kl = pass_kl.back().ptr;
      o.diffs = pass_d.back().ptr;
      o.total = counters.ptr;
      o.cap = cap;
      o.res_off = res_off.ptr;
      o.res_cnt = res_cnt.ptr;
      o.res_pass = res_pass.ptr;
      o.pass = uint8_t(pass);
      o.fail_list = lists[pass & 1].ptr;
      o.fail_count = counters.ptr + 1;
      o.steps = counters.ptr + 2;
      o.next = counters.ptr + 3;
      o.unsorted = counters.ptr + 4;
      o.unsorted_list = unsorted_list.ptr;
      FMG_CK(cudaMemsetAsync(counters.ptr + 4, 0, sizeof(unsigned long long), s));
      const unsigned blocks = unsigned(T / nt);
      CodePatterns cp{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      static const bool trace = std::getenv("FMG_TRACE") != nullptr;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (trace) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, s);
      }
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        if (short_pat)
          k_inexact<true, W><<<blocks, nt, smem, s>>>(ix->view(), cp, list, pending, z, sc, o);
        else
          k_inexact<false, W><<<blocks, nt, smem, s>>>(ix->view(), cp, list, pending, z, sc, o);
      });
      FMG_CK(cudaGetLastError());
      unsigned long long host_ctr[5];
      FMG_CK(cudaMemcpyAsync(host_ctr, counters.ptr, sizeof(host_ctr), cudaMemcpyDeviceToHost, s));
      FMG_CK(cudaStreamSynchronize(s));
      const uint64_t failed = host_ctr[1];
      if (host_ctr[4] > 0) {  // sort this pass's large result sets in place
        k_sort_segments<<<unsigned(host_ctr[4]), 256, 0, s>>>(unsorted_list.ptr, res_off.ptr, res_cnt.ptr,
                                                              pass_kl.back().ptr, pass_d.back().ptr, too_big.ptr);
        FMG_CK(cudaGetLastError());
        uint32_t tb_flag = 0;
        FMG_CK(cudaMemcpyAsync(&tb_flag, too_big.ptr, 4, cudaMemcpyDeviceToHost, s));
        FMG_CK(cudaStreamSynchronize(s));
        if (tb_flag) need_cub_sort = true;
      }
      if (trace) {
        cudaEventRecord(ev1, s);
        cudaEventSynchronize(ev1);
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        unsigned long long st = 0;
        cudaMemcpy(&st, counters.ptr + 2, 8, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[fmg] inexact pass %d: %llu patterns, T=%llu nt=%d S=%u R=%u smem=%zu per_sm=%d: %.3f ms, "
                "%llu failed, %llu steps so far\n", pass, (unsigned long long)pending, (unsigned long long)T, nt, S,
                R, smem, per_sm, ms, (unsigned long long)failed, st);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
      }
      list = lists[pass & 1].ptr;
      if (failed > 0) {
        // grow whichever capacity might have been the cause
        R = std::min<uint32_t>(R * 8, 1u << 22);
        S = std::min<uint32_t>(S_max, S * 2);
        cap = std::max<uint64_t>(cap, std::min<uint64_t>(uint64_t(host_ctr[0]) * 2, 1ull << 31));
        cap = std::max<uint64_t>(cap, failed * uint64_t(R));
        cap = std::min<uint64_t>(cap, 1ull << 31);
      }
      pending = failed;
      // the next pass reads `list` while writing the other list
    }
    static const bool trace_post = std::getenv("FMG_TRACE") != nullptr;
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (trace_post) {
      cudaEventCreate(&pe0);
      cudaEventCreate(&pe1);
      cudaEventRecord(pe0, s);
    }
    // CSR: row_off[q+1] = inclusive sum of counts
    DevBuf<uint64_t> c64(count, s);
    k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, res_cnt.ptr, c64.ptr);
    size_t tmp_bytes = 0;
    FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, c64.ptr, res->row_off + 1, count, s));
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tmp_bytes, c64.ptr, res->row_off + 1, count, s));
    uint64_t total = 0;
    FMG_CK(cudaMemcpyAsync(&total, res->row_off + count, sizeof(total), cudaMemcpyDeviceToHost, s));
    unsigned long long steps = 0;
    FMG_CK(cudaMemcpyAsync(&steps, counters.ptr + 2, sizeof(steps), cudaMemcpyDeviceToHost, s));
    FMG_CK(cudaStreamSynchronize(s));
    const bool unsorted = need_cub_sort;
    res->total = total;
    res->steps = steps;
    FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->k), std::max<uint64_t>(total, 1) * sizeof(uint32_t), s));
    FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->l), std::max<uint64_t>(total, 1) * sizeof(uint32_t), s));
    FMG_CK(cudaMallocAsync(reinterpret_cast<void**>(&res->diffs), std::max<uint64_t>(total, 1), s));
    for (size_t p = 0; p < pass_kl.size(); ++p) {
      k_gather_matches<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, res_off.ptr, res_cnt.ptr, res_pass.ptr,
                                                                     uint8_t(p), pass_kl[p].ptr, pass_d[p].ptr,
                                                                     res->row_off, res->k, res->l, res->diffs);
      FMG_CK(cudaGetLastError());
    }
    if (unsorted && total > 0) {
      // a pattern had more than kSortMax results: segmented sort of everything by (k, l)
      FMG_REQUIRE(total < (1ull << 31), "too many inexact results for one call");
      DevBuf<uint64_t> keys(total, s), keys2(total, s);
      DevBuf<uint8_t> d2(total, s);
      k_pack_keys<<<unsigned((total + 255) / 256), 256, 0, s>>>(total, res->k, res->l, keys.ptr);
      size_t sb = 0;
      FMG_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, keys.ptr, keys2.ptr, res->diffs, d2.ptr, int(total),
                                                 int(count), res->row_off, res->row_off + 1, s));
      DevBuf<uint8_t> stmp(sb, s);
      FMG_CK(cub::DeviceSegmentedSort::SortPairs(stmp.ptr, sb, keys.ptr, keys2.ptr, res->diffs, d2.ptr, int(total),
                                                 int(count), res->row_off, res->row_off + 1, s));
      k_unpack_keys<<<unsigned((total + 255) / 256), 256, 0, s>>>(total, keys2.ptr, d2.ptr, res->k, res->l,
                                                                   res->diffs);
      FMG_CK(cudaGetLastError());
    }
    FMG_CK(cudaStreamSynchronize(s));
    if (trace_post) {
      cudaEventRecord(pe1, s);
      cudaEventSynchronize(pe1);
      float ms = 0;
      cudaEventElapsedTime(&ms, pe0, pe1);
      fprintf(stderr, "[fmg] inexact post (CSR, gather, %s): %.3f ms, %llu results\n",
              unsorted ? "segmented sort" : "no sort", ms, (unsigned long long)total);
      cudaEventDestroy(pe0);
      cudaEventDestroy(pe1);
    }
    return res;
  } catch (...) {
    fmg_matches_free(res);
    throw;
  }
}

// Chunked host-buffer pipeline: H2D, kernel, D2H per chunk on alternating
// streams so the copy engines overlap each other and the kernel.
template <typename Launch>
void pipeline_host(int device, uint64_t count, uint64_t chunk, size_t in_bytes_per, size_t out_bytes_per,
                   const void* host_in, void* host_out, Launch&& launch) {
  constexpr int kSlots = 3;
  cudaStream_t st[kSlots];
  for (int i = 0; i < kSlots; ++i) FMG_CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  std::vector<void*> din(kSlots, nullptr), dout(kSlots, nullptr);
  try {
    for (int i = 0; i < kSlots; ++i) {
      FMG_CK(cudaMallocAsync(&din[i], std::max<size_t>(chunk * in_bytes_per, 1), st[i]));
      FMG_CK(cudaMallocAsync(&dout[i], std::max<size_t>(chunk * out_bytes_per, 1), st[i]));
    }
    uint64_t c = 0;
    for (uint64_t off = 0; off < count; off += chunk, ++c) {
      const int slot = int(c % kSlots);
      const uint64_t len = std::min(chunk, count - off);
      FMG_CK(cudaMemcpyAsync(din[slot], static_cast<const uint8_t*>(host_in) + off * in_bytes_per, len * in_bytes_per,
                             cudaMemcpyHostToDevice, st[slot]));
      launch(din[slot], len, dout[slot], st[slot]);
      FMG_CK(cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + off * out_bytes_per, dout[slot], len * out_bytes_per,
                             cudaMemcpyDeviceToHost, st[slot]));
    }
    for (int i = 0; i < kSlots; ++i) FMG_CK(cudaStreamSynchronize(st[i]));
  } catch (...) {
    for (int i = 0; i < kSlots; ++i) cudaStreamSynchronize(st[i]);
    for (int i = 0; i < kSlots; ++i) {
      if (din[i]) cudaFreeAsync(din[i], st[i]);
      if (dout[i]) cudaFreeAsync(dout[i], st[i]);
      cudaStreamSynchronize(st[i]);
      cudaStreamDestroy(st[i]);
    }
    throw;
  }
  for (int i = 0; i < kSlots; ++i) {
    cudaFreeAsync(din[i], st[i]);
    cudaFreeAsync(dout[i], st[i]);
    cudaStreamSynchronize(st[i]);
    cudaStreamDestroy(st[i]);
  }
}

}  // namespace

extern "C" {

const char* fmg_last_error(void) { return fmg::g_last_error.c_str(); }

int fmg_device_count(int* count) {
  return fmg::guard([&] {
    FMG_REQUIRE(count != nullptr, "null output pointer");
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

int fmg_index_create(int device, const void* bucket_records, uint64_t n_buckets, uint64_t n, uint64_t sentinel_row,
                     const uint64_t c[5], fmg_index** out) {
  return fmg::guard([&] {
    FMG_REQUIRE(out != nullptr && bucket_records != nullptr && c != nullptr, "null argument");
    *out = nullptr;
    FMG_REQUIRE(n >= 1, "index covers an empty reference");
    FMG_REQUIRE(n + 1 < 0xFFFFFFFFull, "reference too long for 32-bit rows");
    FMG_REQUIRE(n_buckets == (n + 1 + 127) / 128, "bucket count does not match n");
    FMG_REQUIRE(sentinel_row <= n, "sentinel row outside [0, n]");
    FMG_REQUIRE(c[0] == 0 && c[4] == n, "C table endpoints wrong");
    for (int s = 0; s < 4; ++s) FMG_REQUIRE(c[s] <= c[s + 1], "C table not non-decreasing");
    int ndev = 0;
    FMG_CK(cudaGetDeviceCount(&ndev));
    FMG_REQUIRE(device >= 0 && device < ndev, "CUDA device ordinal out of range");
    DeviceScope scope(device);
    auto* ix = new fmg_index();
    try {
      ix->device = device;
      ix->n = n;
      ix->sentinel_row = sentinel_row;
      for (int s = 0; s < 5; ++s) ix->c[s] = c[s];
      ix->n_buckets = n_buckets;
      ix->words = choose_words(n_buckets);
      ix->sms = fmg::sm_count(device);
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        ix->n_lines = (n_buckets * 128 + fmg::LineTraits<W>::kChars - 1) / fmg::LineTraits<W>::kChars;
        FMG_CK(cudaMalloc(&ix->lines, ix->n_lines * fmg::LineTraits<W>::kBytes));
        FMG_CK(cudaMalloc(&ix->err, sizeof(uint32_t)));
        FMG_CK(cudaMemset(ix->err, 0, sizeof(uint32_t)));
        uint64_t* staging = nullptr;
        FMG_CK(cudaMalloc(&staging, n_buckets * 64));
        FMG_CK(cudaMemcpy(staging, bucket_records, n_buckets * 64, cudaMemcpyHostToDevice));
        fmg::k_build_lines<W><<<unsigned((ix->n_lines + 255) / 256), 256>>>(staging, n_buckets, ix->lines,
                                                                             ix->n_lines, ix->err);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        cudaFree(staging);
        FMG_CK(e);
      });
      uint32_t bad = 0;
      FMG_CK(cudaMemcpy(&bad, ix->err, sizeof(bad), cudaMemcpyDeviceToHost));
      FMG_REQUIRE(bad == 0, "bucket base does not fit 32 bits");
      // Allow the stream-ordered pool to keep freed blocks (host entry points
      // allocate per call).
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      *out = ix;
    } catch (...) {
      fmg_index_destroy(ix);
      throw;
    }
  });
}

int fmg_index_set_samples(fmg_index* ix, const uint64_t* sa_samples, uint64_t count) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(sa_samples != nullptr, "null argument");
    FMG_REQUIRE(count == ix->n / 32 + 1, "sample count does not match n");
    std::vector<uint32_t> s32(count);
    for (uint64_t i = 0; i < count; ++i) {
      FMG_REQUIRE(sa_samples[i] <= ix->n, "suffix-array sample out of range");
      s32[i] = uint32_t(sa_samples[i]);
    }
    fmg::DeviceScope scope(ix->device);
    if (ix->samples) cudaFree(ix->samples);
    ix->samples = nullptr;
    FMG_CK(cudaMalloc(&ix->samples, count * sizeof(uint32_t)));
    FMG_CK(cudaMemcpy(ix->samples, s32.data(), count * sizeof(uint32_t), cudaMemcpyHostToDevice));
    ix->n_samples = count;
  });
}

int fmg_index_info(const fmg_index* ix, uint64_t* n, int* device, uint64_t* device_bytes) {
  return fmg::guard([&] {
    check_index(ix);
    if (n) *n = ix->n;
    if (device) *device = ix->device;
    if (device_bytes) {
      uint64_t lb = 0;
      with_words(ix, [&](auto wt) { lb = fmg::LineTraits<decltype(wt)::value>::kBytes; });
      *device_bytes = ix->n_lines * lb + ix->n_samples * 4;
    }
  });
}

void fmg_index_destroy(fmg_index* ix) {
  if (!ix) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ix->device);
  if (ix->lines) cudaFree(ix->lines);
  if (ix->samples) cudaFree(ix->samples);
  if (ix->err) cudaFree(ix->err);
  if (prev >= 0) cudaSetDevice(prev);
  delete ix;
}

int fmg_occ_pair(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    launch_occ_pair(ix, kl, count, out, as_stream(stream));
  });
}

// Tuning hook (not part of include/fmgpu.h): same as fmg_occ_pair with an
// explicit pairs-per-thread and block size.
int fmgx_occ_pair_tuned(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, void* stream,
                        int per, int threads) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    launch_occ_pair(ix, kl, count, out, as_stream(stream), per, threads);
  });
}

// Tuning hook: L2 fetch granularity of the current context on `device`
// (cudaLimitMaxL2FetchGranularity; 32 = fetch exactly the 32-byte sector a
// line load needs).  Returns the previous value in *prev.
int fmgx_set_l2_fetch_granularity(int device, int bytes, int* prev) {
  return fmg::guard([&] {
    fmg::DeviceScope scope(device);
    size_t old = 0;
    FMG_CK(cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity));
    if (prev) *prev = int(old);
    if (bytes >= 0) FMG_CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(bytes)));
  });
}

// Measured random 32-byte fetches per second on `device` over `bytes` of
// memory (>> L2), best of 3 launches of `count` reads.  Used by bench.py as
// the request roofline of HBM-resident Occ steps.
int fmgx_random_fetch_rate(int device, uint64_t bytes, uint64_t count, double* rate) {
  return fmg::guard([&] {
    FMG_REQUIRE(rate != nullptr && bytes >= 32 && count > 0, "bad argument");
    fmg::DeviceScope scope(device);
    uint8_t* buf = nullptr;
    unsigned long long* sink = nullptr;
    FMG_CK(cudaMalloc(&buf, bytes));
    FMG_CK(cudaMalloc(&sink, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    cudaError_t err = cudaMemset(buf, 1, bytes);
    for (int r = 0; r < 4 && err == cudaSuccess; ++r) {
      cudaEventRecord(e0);
      fmg::k_random_fetch<<<unsigned((count + 255) / 256), 256>>>(buf, bytes / 32, count, uint64_t(r) * 7919, sink);
      cudaEventRecord(e1);
      err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0) best = std::min(best, ms);  // first launch is warm-up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(sink);
    FMG_CK(err);
    *rate = double(count) / (double(best) * 1e-3);
  });
}

int fmg_occ_pair_host(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 21);
    pipeline_host(ix->device, count, std::max<uint64_t>(chunk, 1), 8, 32, kl, out,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_occ_pair(ix, static_cast<const uint32_t*>(din), len, static_cast<uint32_t*>(dout), s);
                  });
    take_input_error(ix, nullptr, "Occ position out of range or pair out of order");
  });
}

int fmg_exact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count, uint32_t* kl_out,
              void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    launch_exact_codes(ix, codes, offsets, count, kl_out, as_stream(stream), nullptr);
  });
}

int fmg_exact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, uint32_t* kl_out,
                     void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    fmg::DeviceScope scope(ix->device);
    launch_exact_packed(ix, packed, m, count, kl_out, as_stream(stream), nullptr);
  });
}

int fmg_exact_host(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                   uint32_t* kl_out) {
  return fmg::guard([&] {
    check_index(ix);
    if (count == 0) return;
    FMG_REQUIRE(offsets[0] == 0 && offsets[count] >= count, "pattern offsets must start at 0; patterns non-empty");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s;
    FMG_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      DevBuf<uint8_t> dc(offsets[count], s);
      DevBuf<uint64_t> doff(count + 1, s);
      DevBuf<uint32_t> dout(2 * count, s);
      FMG_CK(cudaMemcpyAsync(dc.ptr, codes, offsets[count], cudaMemcpyHostToDevice, s));
      FMG_CK(cudaMemcpyAsync(doff.ptr, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, s));
      validate_patterns_device(dc.ptr, doff.ptr, count, s);
      launch_exact_codes(ix, dc.ptr, doff.ptr, count, dout.ptr, s, nullptr);
      FMG_CK(cudaMemcpyAsync(kl_out, dout.ptr, 2 * count * 4, cudaMemcpyDeviceToHost, s));
      FMG_CK(cudaStreamSynchronize(s));
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  });
}

int fmg_exact_packed_host(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count,
                          uint32_t* kl_out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 22);
    pipeline_host(ix->device, count, chunk, 8, 8, packed, kl_out,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_exact_packed(ix, static_cast<const uint64_t*>(din), m, len, static_cast<uint32_t*>(dout),
                                        s, nullptr);
                  });
  });
}

int fmg_inexact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count, int max_diff,
                fmg_matches** out, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = as_stream(stream);
    const uint64_t max_len = validate_patterns_device(codes, offsets, count, s);
    *out = run_inexact(ix, codes, offsets, count, max_len, max_diff, s);
  });
}

int fmg_inexact_host(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                     int max_diff, fmg_matches** out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
    if (count > 0)
      FMG_REQUIRE(offsets[0] == 0 && offsets[count] >= count, "pattern offsets must start at 0; patterns non-empty");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s;
    FMG_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      DevBuf<uint8_t> dc(count ? offsets[count] : 0, s);
      DevBuf<uint64_t> doff(count + 1, s);
      if (count) {
        FMG_CK(cudaMemcpyAsync(dc.ptr, codes, offsets[count], cudaMemcpyHostToDevice, s));
        FMG_CK(cudaMemcpyAsync(doff.ptr, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, s));
      }
      const uint64_t max_len = validate_patterns_device(dc.ptr, doff.ptr, count, s);
      *out = run_inexact(ix, dc.ptr, doff.ptr, count, max_len, max_diff, s);
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  });
}

int fmg_inexact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, int max_diff,
                       fmg_matches** out, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    fmg::DeviceScope scope(ix->device);
    *out = run_inexact(ix, nullptr, nullptr, count, m, max_diff, as_stream(stream), packed);
  });
}

int fmg_inexact_packed_host(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, int max_diff,
                            fmg_matches** out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s;
    FMG_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    try {
      DevBuf<uint64_t> dp(count, s);
      if (count) FMG_CK(cudaMemcpyAsync(dp.ptr, packed, count * 8, cudaMemcpyHostToDevice, s));
      *out = run_inexact(ix, nullptr, nullptr, count, m, max_diff, s, dp.ptr);
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      throw;
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  });
}

int fmg_matches_size(const fmg_matches* m, uint64_t* total, uint64_t* patterns) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr, "null matches handle");
    if (total) *total = m->total;
    if (patterns) *patterns = m->patterns;
  });
}

int fmg_matches_steps(const fmg_matches* m, uint64_t* steps) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr && steps != nullptr, "null argument");
    *steps = m->steps;
  });
}

int fmg_matches_copy(const fmg_matches* m, uint64_t* row_offsets, uint32_t* k, uint32_t* l, uint8_t* diffs,
                     int to_host) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr, "null matches handle");
    fmg::DeviceScope scope(m->device);
    const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (row_offsets) FMG_CK(cudaMemcpy(row_offsets, m->row_off, (m->patterns + 1) * 8, kind));
    if (m->total) {
      if (k) FMG_CK(cudaMemcpy(k, m->k, m->total * 4, kind));
      if (l) FMG_CK(cudaMemcpy(l, m->l, m->total * 4, kind));
      if (diffs) FMG_CK(cudaMemcpy(diffs, m->diffs, m->total, kind));
    }
  });
}

void fmg_matches_free(fmg_matches* m) {
  if (!m) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  // pool allocations (run_inexact synchronised its stream before returning)
  if (m->row_off) cudaFreeAsync(m->row_off, 0);
  if (m->k) cudaFreeAsync(m->k, 0);
  if (m->l) cudaFreeAsync(m->l, 0);
  if (m->diffs) cudaFreeAsync(m->diffs, 0);
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

int fmg_psi_inverse(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint8_t* out_sym, uint32_t* out_row,
                    void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    with_words(ix, [&](auto wt) {
      fmg::k_psi<decltype(wt)::value><<<unsigned((count + 255) / 256), 256, 0, as_stream(stream)>>>(
          ix->view(), rows, count, out_sym, out_row, ix->err);
    });
    FMG_CK(cudaGetLastError());
  });
}

int fmg_locate_rows(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(ix->samples != nullptr, "index has no suffix-array samples (fmg_index_set_samples)");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    launch_locate(ix, rows, count, out_pos, as_stream(stream));
    FMG_CK(cudaGetLastError());
  });
}

int fmg_locate_rows_host(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(ix->samples != nullptr, "index has no suffix-array samples (fmg_index_set_samples)");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 22);
    pipeline_host(ix->device, count, chunk, 4, 4, rows, out_pos,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_locate(ix, static_cast<const uint32_t*>(din), len, static_cast<uint32_t*>(dout), s);
                    FMG_CK(cudaGetLastError());
                  });
    take_input_error(ix, nullptr, "row out of range");
  });
}

int fmg_stream_sync(void* stream) {
  return fmg::guard([&] { FMG_CK(cudaStreamSynchronize(as_stream(stream))); });
}

}  // extern "C"
