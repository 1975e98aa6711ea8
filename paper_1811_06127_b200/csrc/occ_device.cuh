// Device-side primitives of the Occ step on the line layout.
//
// Layout.  The reference keeps one 128-character bucket per
// 4 x u64 base + 32 packed bytes (index.py:24-36, serialize.py:87-92).  On the
// GPU each bucket is split into two 32-byte LINES of 64 characters:
//
//     struct Line { u32 base[4]; u64 w[2]; }          // 32 B = one DRAM sector
//
// base[s] = occurrences of symbol s strictly before the line in the raw packed
// transform ('$' packed as A, exactly like the reference's bucket bases,
// index.py:83-91); w[0], w[1] hold characters 0..31 and 32..63 of the line in
// the reference's bit order (character j in bits 2j..2j+1, alphabet.py:53-56).
// Any Occ(b, p) therefore reads exactly one 32-byte sector, fetched with one
// 256-bit load (LDG.E.ENL2.256).
//
// In-line rank by masked popcount (the GPU-native form of the paper's nibble
// pipeline, kernels.py:161-211): with lo = w & 0x55.., hi = (w >> 1) & 0x55..
// and a mask M of the fields 0..r,
//     T = popc(lo & hi & M)      G = popc(hi & M) - T
//     C = popc(lo & M) - T       A = (r + 1) - popc(hi & M) - popc(lo & M) + T
// The A lane then drops the terminator once p >= sentinel_row (occ.py:39-40,
// 54-55, 92-95).
#pragma once

#include <cstdint>

namespace fmg {

struct __align__(32) Line {
  uint32_t base[4];
  uint64_t w[2];
};
static_assert(sizeof(Line) == 32, "line must be one 32-byte sector");

// Everything a kernel needs about the index, passed by value (kernel params
// live in the constant bank, so C[] is a constant-cache broadcast).
struct IndexView {
  const Line* lines;
  const uint32_t* samples;  // suffix-array rows 0, 32, 64, ... (may be null)
  uint32_t n;
  uint32_t sentinel_row;
  uint32_t c[5];
};

constexpr uint64_t kFieldLo = 0x5555555555555555ull;

// One 256-bit read-only load of a line.  kStream selects L1::no_allocate for
// gathers without reuse (Occ microbenchmark); search kernels keep L1
// allocation so the hot top-of-BWT lines every query starts from are L1 hits.
template <bool kStream>
__device__ __forceinline__ void load_line(const Line* p, uint32_t b[4], uint64_t w[2]) {
  uint64_t a0, a1, a2, a3;
  if (kStream) {
    asm("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
        : "l"(p));
  } else {
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
        : "l"(p));
  }
  b[0] = uint32_t(a0);
  b[1] = uint32_t(a0 >> 32);
  b[2] = uint32_t(a1);
  b[3] = uint32_t(a1 >> 32);
  w[0] = a2;
  w[1] = a3;
}

// Masks of the 2-bit fields 0..r (inclusive) of a 64-field line.
__device__ __forceinline__ void prefix_masks(uint32_t r, uint64_t& m0, uint64_t& m1) {
  m0 = ~0ull >> (62u - 2u * min(r, 31u));
  m1 = (r >= 32u) ? (~0ull >> (126u - 2u * r)) : 0ull;
}

// Counts of A, C, G, T among fields 0..r of the line (raw: '$' counts as A).
__device__ __forceinline__ void count4(const uint64_t w[2], uint32_t r, uint32_t out[4]) {
  uint64_t m0, m1;
  prefix_masks(r, m0, m1);
  const uint64_t lo0 = w[0] & kFieldLo & m0, hi0 = (w[0] >> 1) & kFieldLo & m0;
  const uint64_t lo1 = w[1] & kFieldLo & m1, hi1 = (w[1] >> 1) & kFieldLo & m1;
  const uint32_t t = __popcll(lo0 & hi0) + __popcll(lo1 & hi1);
  const uint32_t h = __popcll(hi0) + __popcll(hi1);
  const uint32_t l = __popcll(lo0) + __popcll(lo1);
  out[3] = t;
  out[2] = h - t;
  out[1] = l - t;
  out[0] = r + 1u - h - l + t;
}

// Count of one symbol among fields 0..r of the line (raw).
__device__ __forceinline__ uint32_t count1(const uint64_t w[2], uint32_t r, uint32_t sym) {
  uint64_t m0, m1;
  prefix_masks(r, m0, m1);
  const uint64_t rep = uint64_t(sym) * kFieldLo;  // sym replicated in every field
  uint64_t x0 = ~(w[0] ^ rep), x1 = ~(w[1] ^ rep);
  x0 = x0 & (x0 >> 1) & kFieldLo & m0;
  x1 = x1 & (x1 >> 1) & kFieldLo & m1;
  return __popcll(x0) + __popcll(x1);
}

// Symbol stored at field r of the line.
__device__ __forceinline__ uint32_t field_at(const uint64_t w[2], uint32_t r) {
  const uint64_t word = (r < 32u) ? w[0] : w[1];
  return uint32_t((word >> ((r & 31u) << 1)) & 3ull);
}

// All four Occ(b, p) for 0 <= p <= n given the line holding p.
__device__ __forceinline__ void occ4_from_line(const IndexView& ix, const uint32_t b[4],
                                               const uint64_t w[2], uint32_t p, uint32_t out[4]) {
  uint32_t in[4];
  count4(w, p & 63u, in);
  out[0] = b[0] + in[0] - (p >= ix.sentinel_row ? 1u : 0u);
  out[1] = b[1] + in[1];
  out[2] = b[2] + in[2];
  out[3] = b[3] + in[3];
}

// a[i] for a runtime i without forcing the array into local memory.
__device__ __forceinline__ uint32_t sel4(const uint32_t a[4], uint32_t i) {
  return i == 0u ? a[0] : i == 1u ? a[1] : i == 2u ? a[2] : a[3];
}
__device__ __forceinline__ uint32_t c_of(const IndexView& ix, uint32_t s) {
  return s == 0u ? ix.c[0] : s == 1u ? ix.c[1] : s == 2u ? ix.c[2] : s == 3u ? ix.c[3] : ix.c[4];
}

// Occ(sym, p) for 0 <= p <= n given the line holding p.
__device__ __forceinline__ uint32_t occ1_from_line(const IndexView& ix, const uint32_t b[4],
                                                   const uint64_t w[2], uint32_t p, uint32_t sym) {
  uint32_t v = sel4(b, sym) + count1(w, p & 63u, sym);
  if (sym == 0u && p >= ix.sentinel_row) v -= 1u;
  return v;
}

// The eight values of an Occ step at (k-1, l): lo[] = Occ(., k-1), hi[] =
// Occ(., l).  k == 0 gives lo = 0 (occ.py:74-77); the root interval (0, n)
// needs no memory at all (Occ(b, n) = c[b+1] - c[b]).  When both ends share a
// line it is fetched once (occ.py:86-96 does the same per bucket).
template <bool kStream>
__device__ __forceinline__ void occ_step(const IndexView& ix, uint32_t k, uint32_t l,
                                         uint32_t lo[4], uint32_t hi[4]) {
  if (k == 0u && l == ix.n) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      lo[s] = 0u;
      hi[s] = ix.c[s + 1] - ix.c[s];
    }
    return;
  }
  uint32_t bh[4], bl[4];
  uint64_t wh[2], wl[2];
  const uint32_t lh = l >> 6;
  load_line<kStream>(ix.lines + lh, bh, wh);
  const bool has_low = k != 0u;
  const uint32_t low = k - 1u;
  const uint32_t ll = has_low ? (low >> 6) : lh;
  if (ll != lh) {
    load_line<kStream>(ix.lines + ll, bl, wl);
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) bl[s] = bh[s];
    wl[0] = wh[0];
    wl[1] = wh[1];
  }
  occ4_from_line(ix, bh, wh, l, hi);
  if (has_low) {
    occ4_from_line(ix, bl, wl, low, lo);
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) lo[s] = 0u;
  }
}

}  // namespace fmg
