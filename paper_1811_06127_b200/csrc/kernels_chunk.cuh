// Chunk layout and Occ-step kernel for HBM-resident indexes (occ.py:59-96).
//
// B200 serves a random L2 miss with a 128-byte DRAM fetch (measured:
// tools/micro/l2pin.cu, profiles/r02_occ_layout.md), so for an index that
// lives in HBM the cost of an Occ step is the number of distinct 128-byte
// chunks it touches, and every byte of a chunk should be BWT characters.
// The 32-byte-line layout (occ_device.cuh, W = 2) spends half of each line on
// its checkpoint: 256 characters per 128-byte fetch.  This layout packs 416:
//
//   chunk j = 128 bytes = 4 sectors of 8 x u32 (little-endian), characters
//   416j .. 416j + 415 of the transform ('$' stored as A, reference bit
//   order: character t of a u32 word in bits 2t..2t+1):
//     sector 0: u32[0..2] = C, G, T occurrences in [0, 416j) (raw: '$' is
//               counted as A, exactly like the reference's bucket bases,
//               index.py:83-91); u32[3..7] = characters 0..79
//     sector s = 1..3: u32[0] = C | G << 10 | T << 20, the occurrences in
//               characters [0, 80 + 112(s-1)) of the chunk;
//               u32[1..7] = characters 80 + 112(s-1) .. + 111
//
// Occ(b, p) needs sector 0 of p's chunk (the base) and the sector holding p
// (the delta and the characters), both inside one 128-byte fetch, and counts
// at most 112 characters (two interleaved word pairs, six popcounts).  A is
// never stored: raw A = p + 1 - C - G - T, minus one once p >= sentinel_row
// (occ.py:39-40, 54-55, 92-95).  Counts are u32: n + 1 < 2^32.
#pragma once

#include <cstdint>

#include "occ_device.cuh"

namespace fmg {

// NS sectors per chunk: 4 (128 bytes, 416 characters; the DRAM fetch
// granularity) or 2 (64 bytes, 192 characters: the first two sectors of the
// same format, read with the L2::64B fetch hint so a miss moves 64 bytes).
template <int NS>
struct ChunkTraits {
  static_assert(NS == 2 || NS == 4, "2 or 4 sectors per chunk");
  static constexpr uint32_t kChars = NS == 4 ? 416u : 192u;
  static constexpr uint32_t kBytes = 32u * NS;
  static constexpr uint32_t kWords = 8u * NS;  // u32
};

// first character of sector s inside its chunk, and its data field offset
// inside the sector's 128 two-bit fields
__host__ __device__ constexpr uint32_t chunk_sector_start(uint32_t s) { return s == 0 ? 0u : 80u + 112u * (s - 1u); }

__device__ __forceinline__ uint32_t chunk_sector_of(uint32_t r) {
  // r in [0, 416): 0 for r < 80, else 1 + (r - 80) / 112 (a constant
  // divisor: the compiler emits a multiply-high)
  return r < 80u ? 0u : 1u + (r - 80u) / 112u;
}

// Build: bucket records (4 x u64 LE base + 32 B chars per 128 characters,
// serialize.py:87-92) -> chunks.  One thread per chunk.
template <int NS>
__global__ void k_build_chunks(const uint64_t* __restrict__ rec, uint64_t nb, uint32_t* __restrict__ chunks,
                               uint64_t n_chunks, uint32_t* __restrict__ err) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n_chunks) return;
  const uint64_t c0 = j * ChunkTraits<NS>::kChars;  // multiple of 32: a word boundary of its bucket
  const uint64_t b0 = c0 >> 7;
  const uint64_t* r = rec + b0 * 8;
  uint32_t cgt[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (r[1 + s] >= 0xFFFFFFFFull && err) atomicOr(err, 1u);
    cgt[s] = uint32_t(r[1 + s]);
  }
  // characters of the bucket before c0 (whole 32-char words)
  const uint32_t skip = uint32_t((c0 & 127u) >> 5);
  for (uint32_t q = 0; q < skip; ++q) {
    const uint64_t w = r[4 + q], lo = w & kFieldLo, hi = (w >> 1) & kFieldLo;
    const uint32_t t = __popcll(lo & hi);
    cgt[0] += __popcll(lo) - t;
    cgt[1] += __popcll(hi) - t;
    cgt[2] += t;
  }
  // the 26 data words of 16 characters each, in chunk order
  auto word16 = [&](uint64_t c) -> uint32_t {  // characters c .. c+15 (c multiple of 16)
    const uint64_t b = c >> 7;
    if (b >= nb) return 0u;
    const uint32_t* chars = reinterpret_cast<const uint32_t*>(rec + b * 8 + 4);
    return chars[(c & 127u) >> 4];
  };
  uint32_t out[8 * NS];
  out[0] = cgt[0];
  out[1] = cgt[1];
  out[2] = cgt[2];
  uint32_t dc = 0, dg = 0, dt = 0;  // running counts inside the chunk
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t first = s == 0 ? 3u : 1u;
    if (s > 0) out[8 * s] = dc | (dg << 10) | (dt << 20);
#pragma unroll
    for (uint32_t q = first; q < 8; ++q) {
      const uint32_t w = word16(c0 + chunk_sector_start(uint32_t(s)) + 16u * (q - first));
      out[8 * s + q] = w;
      const uint32_t lo = w & 0x55555555u, hi = (w >> 1) & 0x55555555u, t = __popc(lo & hi);
      dc += __popc(lo) - t;
      dg += __popc(hi) - t;
      dt += t;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(chunks + j * ChunkTraits<NS>::kWords);
#pragma unroll
  for (int q = 0; q < 2 * NS; ++q) dst[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
}

// C, G, T among the sector's data fields up to and including chunk character
// r (sector s = sector of r).  v = the sector's 4 u64 words.
__device__ __forceinline__ void chunk_count3(const uint64_t v[4], uint32_t s, uint32_t r, uint32_t& c, uint32_t& g,
                                             uint32_t& t) {
  // field index of r inside the sector's 128 fields: data starts at field 48
  // (sector 0, after three u32) or 16 (after one u32)
  const uint32_t f0 = s == 0 ? 48u : 16u;
  const uint32_t f = f0 + r - chunk_sector_start(s);
  uint32_t tt = 0, hh = 0, ll = 0;
#pragma unroll
  for (int k = 0; k < 4; k += 2) {
    // fields [f0, f] of words k, k+1
    const uint64_t m0 = word_mask(f, k) & ~word_mask(f0 - 1u, k);
    const uint64_t m1 = word_mask(f, k + 1) & ~word_mask(f0 - 1u, k + 1);
    const uint64_t x0 = v[k] & m0, x1 = v[k + 1] & m1;
    const uint64_t lo = (x0 & kFieldLo) | ((x1 & kFieldLo) << 1);
    const uint64_t hi = ((x0 >> 1) & kFieldLo) | (x1 & ~kFieldLo);
    tt += __popcll(lo & hi);
    hh += __popcll(hi);
    ll += __popcll(lo);
  }
  t = tt;
  g = hh - tt;
  c = ll - tt;
}

// Sector s of chunk j, predicated (no request when !go).  Two-sector chunks
// carry the L2::64B hint: the miss fetches the 64-byte chunk, not 128 bytes.
// `wide` (two-sector chunks only): the step's two chunks are the halves of one
// 128-byte line, so the loads go without the hint and ONE 128-byte fetch
// serves both ends instead of two 64-byte ones.
template <int NS>
__device__ __forceinline__ void ld_sector_pred(bool go, const uint32_t* chunks, uint64_t j, uint32_t s,
                                               uint64_t v[4], bool wide = false) {
  const uint32_t* p = chunks + j * ChunkTraits<NS>::kWords + 8 * s;
  if constexpr (NS == 2) {
    asm volatile(
        "{\n\t.reg .pred q, w;\n\tsetp.ne.u32 q, %4, 0;\n\tsetp.ne.u32 w, %6, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%5];\n\t"
        "@w ld.global.nc.L1::no_allocate.L2::128B.v4.u64 {%0,%1,%2,%3}, [%5];\n\t}"
        : "+l"(v[0]), "+l"(v[1]), "+l"(v[2]), "+l"(v[3])
        : "r"(uint32_t(go && !wide)), "l"(p), "r"(uint32_t(go && wide)));
  } else {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%5];\n\t}"
        : "+l"(v[0]), "+l"(v[1]), "+l"(v[2]), "+l"(v[3])
        : "r"(uint32_t(go)), "l"(p));
  }
}

// Occ(., p) for 0 <= p <= n from sector 0 (h) and p's own sector (d; equal
// to h when p lies in sector 0).
template <int NS>
__device__ __forceinline__ void chunk_occ4(const IndexView& ix, const uint64_t h[4], const uint64_t d[4], uint32_t p,
                                           uint32_t j, uint32_t out[4]) {
  const uint32_t r = p - j * ChunkTraits<NS>::kChars;
  const uint32_t s = chunk_sector_of(r);
  uint32_t c, g, t;
  chunk_count3(d, s, r, c, g, t);
  const uint32_t delta = uint32_t(d[0]);  // sector s >= 1: packed in-chunk counts before the sector
  if (s != 0u) {
    c += delta & 0x3FFu;
    g += (delta >> 10) & 0x3FFu;
    t += (delta >> 20) & 0x3FFu;
  }
  c += uint32_t(h[0]);
  g += uint32_t(h[0] >> 32);
  t += uint32_t(h[1]);
  out[1] = c;
  out[2] = g;
  out[3] = t;
  out[0] = p + 1u - c - g - t - (p >= ix.sentinel_row ? 1u : 0u);
}

// One thread per Occ step.  All sector loads of the step are issued before
// any counting (up to four: the base sector and the character sector of each
// end, each predicated off when it is already loaded), so a warp keeps
// ~2.5 random 32-byte requests per step in flight against one or two
// 128-byte DRAM fetches.
template <int NS>
__global__ void __launch_bounds__(256) k_occ_pair_chunk(IndexView ix, const uint32_t* __restrict__ chunks,
                                                        const uint2* __restrict__ kl, uint64_t count,
                                                        uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint2 q = ld_stream_u2(kl + i);
  const uint32_t k = q.x, l = q.y;
  const bool ok = l <= ix.n && k <= l + 1u;
  if (!ok && err) atomicOr(err, 1u);
  const uint32_t hp = ok ? l : 0u;
  const bool has_low = ok && k != 0u;
  const uint32_t lp = has_low ? k - 1u : hp;
  constexpr uint32_t kC = ChunkTraits<NS>::kChars;
  const uint32_t jh = hp / kC, jl = lp / kC;
  const uint32_t sh = chunk_sector_of(hp - jh * kC), sl = chunk_sector_of(lp - jl * kC);
  uint64_t h_hi[4] = {0, 0, 0, 0}, d_hi[4] = {0, 0, 0, 0}, h_lo[4] = {0, 0, 0, 0}, d_lo[4] = {0, 0, 0, 0};
  const bool other = jl != jh;
#ifndef FMG_CHUNK2_WIDE
// 1: when the step's two 64-byte chunks are the halves of one 128-byte line,
// load them without the 64-byte hint (one 128-byte fetch instead of two
// 64-byte ones).  Measured on config 1-H: 31.9 G steps/s against 38.25 G with
// every load hinted (profiles/r02_ab_1h_chunk2_wide.log) — off.
#define FMG_CHUNK2_WIDE 0
#endif
  const bool wide = NS == 2 && FMG_CHUNK2_WIDE && other && (jl >> 1) == (jh >> 1);
  ld_sector_pred<NS>(true, chunks, jh, 0, h_hi, wide);
  ld_sector_pred<NS>(sh != 0u, chunks, jh, sh, d_hi, wide);
  ld_sector_pred<NS>(other, chunks, jl, 0, h_lo, wide);
  ld_sector_pred<NS>(sl != 0u && (other || sl != sh), chunks, jl, sl, d_lo, wide);
  // resolve aliases: the low end shares whatever the high end loaded
#pragma unroll
  for (int z = 0; z < 4; ++z) {
    if (sh == 0u) d_hi[z] = h_hi[z];
    if (!other) h_lo[z] = h_hi[z];
    d_lo[z] = sl == 0u ? h_lo[z] : ((!other && sl == sh) ? d_hi[z] : d_lo[z]);
  }
  uint32_t lo4[4] = {0u, 0u, 0u, 0u}, hi4[4] = {0u, 0u, 0u, 0u};
  if (ok) chunk_occ4<NS>(ix, h_hi, d_hi, hp, jh, hi4);
  if (has_low) chunk_occ4<NS>(ix, h_lo, d_lo, lp, jl, lo4);
  st_stream_256(out + i * 8, lo4, hi4);
}

}  // namespace fmg
