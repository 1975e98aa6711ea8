// Device-side primitives of the Occ step on the line layout.
//
// Layout.  The reference keeps one 128-character bucket per
// 4 x u64 base + 32 packed bytes (index.py:24-36, serialize.py:87-92).  On the
// GPU the transform is re-cut into LINES of W 64-bit words (32 characters
// each), every line carrying its own checkpoint:
//
//     template <int W> struct Line { u32 base[4]; u64 w[W]; }   // 16 + 8W bytes
//
//   W = 2  : 32 B,   64 chars — one 32-byte sector per Occ (L2-resident indexes)
//   W = 6  : 64 B,  192 chars — two lines per 128-byte DRAM fetch
//   W = 14 : 128 B, 448 chars — one line per 128-byte DRAM fetch
//
// base[s] = occurrences of symbol s strictly before the line in the raw packed
// transform ('$' packed as A, exactly like the reference's bucket bases,
// index.py:83-91); w[] holds the line's characters in the reference's bit
// order (character j in bits 2j..2j+1 of its word, alphabet.py:53-56).  Any
// Occ(b, p) reads one line, with 256-bit loads (LDG.E.ENL2.256), predicated so
// only the sectors up to p are fetched.  B200 serves a random miss with a
// 128-byte DRAM fetch (measured, tools/micro/gather.cu), so for HBM-resident
// indexes the characters per 128 bytes decide throughput; for L2-resident
// ones the sectors per Occ do.  The host picks W by index size.
//
// In-line rank by masked popcount (the GPU-native form of the paper's nibble
// pipeline, kernels.py:161-211): with lo = w & 0x55.., hi = (w >> 1) & 0x55..
// and a mask M of the fields 0..r,
//     T = popc(lo & hi & M)      G = popc(hi & M) - T
//     C = popc(lo & M) - T       A = (r + 1) - popc(hi & M) - popc(lo & M) + T
// Two words are interleaved (even/odd bits) so each word pair costs three
// 64-bit popcounts.  The A lane then drops the terminator once
// p >= sentinel_row (occ.py:39-40, 54-55, 92-95).
#pragma once

#include <cstdint>

namespace fmg {

template <int W>
struct __align__(16) Line {
  uint32_t base[4];
  uint64_t w[W];
};
static_assert(sizeof(Line<2>) == 32, "W=2 line must be one 32-byte sector");
static_assert(sizeof(Line<6>) == 64, "W=6 line must be 64 bytes");
static_assert(sizeof(Line<14>) == 128, "W=14 line must be 128 bytes");

template <int W>
struct LineTraits {
  static constexpr uint32_t kChars = 32u * W;
  static constexpr uint32_t kBytes = 16u + 8u * W;
};

// Everything a kernel needs about the index, passed by value (kernel params
// live in the constant bank, so C[] is a constant-cache broadcast).
struct IndexView {
  const uint8_t* lines;
  const uint32_t* samples;  // suffix-array rows 0, 32, 64, ... (may be null)
  uint32_t n;
  uint32_t sentinel_row;
  uint32_t c[5];
};

constexpr uint64_t kFieldLo = 0x5555555555555555ull;

#ifndef FMG_SEARCH_L2_64B
// 1: the search kernels' line and table loads carry the L2::64B hint, so a
// miss fetches 64 bytes from DRAM instead of 128 (a dependent search step
// uses one 32-byte line).  Measured on B200: config 4 exact 12.44 -> 13.30 G
// seeds/s (it is DRAM-saturated at 128-byte fetches), config 3 z = 1 130.8
// -> 129.9 ms per 14M seeds (latency-bound).  0 restores plain loads (A/B).
#define FMG_SEARCH_L2_64B 1
#endif

// kStream: 0 = default caching; 1 = L1::no_allocate (gathers without reuse);
// 2 = L2 evict_first (lines that must not push a hot working set — the
// prefix table — out of L2).
template <int kStream>
__device__ __forceinline__ void ld256(const uint8_t* p, uint64_t& a0, uint64_t& a1, uint64_t& a2, uint64_t& a3) {
  if (kStream == 1) {
    asm("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
        : "l"(p));
  } else if (kStream == 2) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm("ld.global.nc.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3)
        : "l"(p), "l"(pol));
  } else {
#if FMG_SEARCH_L2_64B
    asm("ld.global.nc.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p));
#else
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p));
#endif
  }
}

// Line index and offset of transform position p.
template <int W>
__device__ __forceinline__ uint32_t line_of(uint32_t p) {
  return p / LineTraits<W>::kChars;  // constant divisor: shift for W=2, mul-hi otherwise
}

// Load line j, fetching only the 32-byte sectors that hold fields 0..r.
// kStream selects L1::no_allocate for gathers without reuse (Occ
// microbenchmark); search kernels keep L1 allocation so the hot top-of-BWT
// lines every query starts from are L1 hits.
template <int W, int kStream>
__device__ __forceinline__ void load_line(const IndexView& ix, uint32_t j, uint32_t rmax, uint32_t b[4],
                                          uint64_t w[W]) {
  const uint8_t* p = ix.lines + size_t(j) * LineTraits<W>::kBytes;
  uint64_t a0, a1, a2, a3;
  ld256<kStream>(p, a0, a1, a2, a3);
  b[0] = uint32_t(a0);
  b[1] = uint32_t(a0 >> 32);
  b[2] = uint32_t(a1);
  b[3] = uint32_t(a1 >> 32);
  w[0] = a2;
  w[1] = a3;
#pragma unroll
  for (int k = 2; k < W; k += 4) {
    if (rmax >= 32u * k) {
      ld256<kStream>(p + 16 + 8 * k, w[k], w[k + 1], w[k + 2], w[k + 3]);
    } else {
      w[k] = w[k + 1] = w[k + 2] = w[k + 3] = 0;
    }
  }
}

#ifndef FMG_OCC_PRED_LOW
#define FMG_OCC_PRED_LOW 1  // occ_step (W = 2): predicated low-line load
#endif

// W = 2 line load issued only when `go` (a predicated-off load makes no
// memory request and keeps the straight-line code of the step).
__device__ __forceinline__ void ld256_pred(bool go, const uint8_t* p, uint64_t& a0, uint64_t& a1, uint64_t& a2,
                                           uint64_t& a3) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
#if FMG_SEARCH_L2_64B
      "@q ld.global.nc.L2::64B.v4.u64 {%0,%1,%2,%3}, [%5];\n\t}"
#else
      "@q ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%5];\n\t}"
#endif
      : "+l"(a0), "+l"(a1), "+l"(a2), "+l"(a3)
      : "r"(uint32_t(go)), "l"(p));
}

// Mask of the fields of word k that lie in 0..r.
// Branch-free: PTX clamps shift counts above 64 (all fields out -> 0).
__device__ __forceinline__ uint64_t word_mask(uint32_t r, int k) {
  const int s = max(62 - 2 * (int(r) - 32 * k), 0);
  uint64_t m;
  asm("shr.b64 %0, %1, %2;" : "=l"(m) : "l"(~0ull), "r"(s));
  return m;
}

// Counts of A, C, G, T among fields 0..r of the line (raw: '$' counts as A).
template <int W>
__device__ __forceinline__ void count4(const uint64_t w[W], uint32_t r, uint32_t out[4]) {
  uint32_t t = 0, h = 0, l = 0;
#pragma unroll
  for (int k = 0; k < W; k += 2) {
    const uint64_t x0 = w[k] & word_mask(r, k), x1 = w[k + 1] & word_mask(r, k + 1);
    const uint64_t lo = (x0 & kFieldLo) | ((x1 & kFieldLo) << 1);
    const uint64_t hi = ((x0 >> 1) & kFieldLo) | (x1 & ~kFieldLo);
    t += __popcll(lo & hi);
    h += __popcll(hi);
    l += __popcll(lo);
  }
  out[3] = t;
  out[2] = h - t;
  out[1] = l - t;
  out[0] = r + 1u - h - l + t;
}

// Count of one symbol among fields 0..r of the line (raw).
template <int W>
__device__ __forceinline__ uint32_t count1(const uint64_t w[W], uint32_t r, uint32_t sym) {
  const uint64_t rep = uint64_t(sym) * kFieldLo;  // sym replicated in every field
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < W; k += 2) {
    uint64_t x0 = ~(w[k] ^ rep), x1 = ~(w[k + 1] ^ rep);
    x0 = x0 & (x0 >> 1) & kFieldLo & word_mask(r, k);       // matches on even bits
    x1 = x1 & (x1 << 1) & ~kFieldLo & word_mask(r, k + 1);  // matches on odd bits
    c += __popcll(x0 | x1);
  }
  return c;
}

// Symbol stored at field r of the line.
template <int W>
__device__ __forceinline__ uint32_t field_at(const uint64_t w[W], uint32_t r) {
  // branch-free select (a plain `w[r >> 5]` would spill w[] to local memory)
  const uint32_t q = r >> 5;
  uint64_t word = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) word |= w[k] & (0ull - uint64_t(q == uint32_t(k)));
  return uint32_t((word >> ((r & 31u) << 1)) & 3ull);
}

// Predicated select (SEL, never a branch): the selects below sit on the
// dependent chain of every Occ step, where a branchy ?: chain cost ~100 of
// the ~800 cycles of an exact-search step (tools/exact_latency.py,
// tools/micro/chase.cu: an L2 hit is ~310 cycles).
__device__ __forceinline__ uint32_t selp32(bool c, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(c)), "r"(a), "r"(b));
  return r;
}

// a[i] for a runtime i in 0..3 without forcing the array into local memory.
__device__ __forceinline__ uint32_t sel4(const uint32_t a[4], uint32_t i) {
  const uint32_t lo = selp32(i & 1u, a[1], a[0]), hi = selp32(i & 1u, a[3], a[2]);
  return selp32(i & 2u, hi, lo);
}
// C[s] for s in 0..4.
__device__ __forceinline__ uint32_t c_of(const IndexView& ix, uint32_t s) {
  const uint32_t lo = selp32(s & 1u, ix.c[1], ix.c[0]), hi = selp32(s & 1u, ix.c[3], ix.c[2]);
  return selp32(s & 4u, ix.c[4], selp32(s & 2u, hi, lo));
}

// All four Occ(b, p) for 0 <= p <= n given the line holding p.
template <int W>
__device__ __forceinline__ void occ4_from_line(const IndexView& ix, const uint32_t b[4], const uint64_t w[W],
                                               uint32_t p, uint32_t r, uint32_t out[4]) {
  uint32_t in[4];
  count4<W>(w, r, in);
  out[0] = b[0] + in[0] - (p >= ix.sentinel_row ? 1u : 0u);
  out[1] = b[1] + in[1];
  out[2] = b[2] + in[2];
  out[3] = b[3] + in[3];
}

// Occ(sym, p) for 0 <= p <= n given the line holding p.
template <int W>
__device__ __forceinline__ uint32_t occ1_from_line(const IndexView& ix, const uint32_t b[4], const uint64_t w[W],
                                                   uint32_t p, uint32_t r, uint32_t sym) {
  uint32_t v = sel4(b, sym) + count1<W>(w, r, sym);
  if (sym == 0u && p >= ix.sentinel_row) v -= 1u;
  return v;
}

// The eight values of an Occ step at (k-1, l): lo[] = Occ(., k-1), hi[] =
// Occ(., l).  k == 0 gives lo = 0 (occ.py:74-77); the root interval (0, n)
// needs no memory at all (Occ(b, n) = c[b+1] - c[b]).  When both ends share a
// line it is fetched once (occ.py:86-96 does the same per bucket).
template <int W, int kStream>
__device__ __forceinline__ uint32_t occ_step(const IndexView& ix, uint32_t k, uint32_t l, uint32_t lo[4],
                                             uint32_t hi[4]) {
  if (k == 0u && l == ix.n) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      lo[s] = 0u;
      hi[s] = ix.c[s + 1] - ix.c[s];
    }
    return 0u;
  }
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint32_t jh = line_of<W>(l), rh = l - jh * kC;
  const bool has_low = k != 0u;
  const uint32_t low = k - 1u;
  const uint32_t jl = has_low ? line_of<W>(low) : jh;
  const uint32_t rl = has_low ? low - jl * kC : 0u;
  // Branch-free: the low line is loaded unconditionally (the same line again
  // — an L1 hit — when k-1 and l share it), so lanes taking one or two lines
  // never split the warp and both counts run as one straight-line block.
  uint32_t bh[4], bl[4];
  uint64_t wh[W], wl[W];
  load_line<W, kStream>(ix, jh, rh, bh, wh);
  if constexpr (W == 2 && kStream == 0 && FMG_OCC_PRED_LOW) {
    // predicated: no second request when both ends share the line
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
    load_line<W, kStream>(ix, jl, rl, bl, wl);
  }
  occ4_from_line<W>(ix, bl, wl, low, rl, lo);
  occ4_from_line<W>(ix, bh, wh, l, rh, hi);
#pragma unroll
  for (int s = 0; s < 4; ++s) lo[s] = has_low ? lo[s] : 0u;
  return jl != jh ? 2u : 1u;  // lines fetched
}

// Work counters (reporting only; the pointer is null on production calls).
// A thread accumulates one u64: Occ steps in the high half, lines fetched in
// the low half; flush_work adds them warp-reduced into ctr[0] (steps) and
// ctr[1] (lines), so a launch costs a handful of same-address atomics.
__device__ __forceinline__ uint64_t work_unit(uint32_t lines) { return (1ull << 32) | lines; }

__device__ __forceinline__ void flush_work(unsigned long long* ctr, uint64_t v) {
  if (ctr == nullptr) return;
  const unsigned mask = __activemask();
  const unsigned st = __reduce_add_sync(mask, unsigned(v >> 32));
  const unsigned ln = __reduce_add_sync(mask, unsigned(v));
  if ((threadIdx.x & 31u) == unsigned(__ffs(mask) - 1)) {
    atomicAdd(ctr, (unsigned long long)st);
    atomicAdd(ctr + 1, (unsigned long long)ln);
  }
}

}  // namespace fmg
