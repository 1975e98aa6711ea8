// Bucket-level rank kernels: the reference's per-bucket plugin surface
// (kernels.py:125-292) as batched sm_100a kernels.  A bucket is 32 packed
// bytes = 128 two-bit fields in the reference's bit order (field j in bits
// 2j..2j+1 of byte j/4, alphabet.py:53-56); a query is (bucket, prefix_len in
// [0, 128], symbol).  Two independent GPU methods:
//
//   method 0 (serves scalar / bytelut / auto): masked popcount over the four
//            words (the same arithmetic as the Occ-step kernels, count4 /
//            count1 in occ_device.cuh);
//   method 1 (serves nibble / simd): the paper's three-phase half-byte
//            pipeline (kernels.py:161-211) mapped onto GPU byte instructions:
//            phase 1 looks every nibble up in the 16-entry tables with byte
//            permutes (PRMT), phase 2 shifts by 2*symbol and tops up / masks
//            the bytes, phase 3 sums |lo - hi| per 8-byte group with the
//            4-byte SAD instruction (__vsadu4); count = 8160 - SAD total,
//            minus the masked padding for A (kernels.py:206, 272).
//
// k_bucket_nibble_trace records the pipeline's intermediate words exactly as
// the reference's KernelTrace does (kernels.py:101-115).
#pragma once

#include <cstdint>

#include "occ_device.cuh"

namespace fmg {

// NibbleTables (kernels.py:53-77): hi[v] packs the counts of each symbol s
// among the two fields of nibble v into bits 2s..2s+1; lo[v] = ~hi[v].
// Bytes v = 0..15 little-endian in four words each.
struct NibbleLut {
  uint32_t lo[4], hi[4];
};

__host__ __device__ constexpr uint32_t nib_hi_byte(uint32_t v) {
  return (1u << ((v & 3u) << 1)) + (1u << (((v >> 2) & 3u) << 1));
}
__host__ __device__ constexpr uint32_t nib_word(uint32_t v0, bool lo) {
  return lo ? ((~nib_hi_byte(v0) & 0xFFu) | ((~nib_hi_byte(v0 + 1) & 0xFFu) << 8) |
               ((~nib_hi_byte(v0 + 2) & 0xFFu) << 16) | ((~nib_hi_byte(v0 + 3) & 0xFFu) << 24))
            : (nib_hi_byte(v0) | (nib_hi_byte(v0 + 1) << 8) | (nib_hi_byte(v0 + 2) << 16) |
               (nib_hi_byte(v0 + 3) << 24));
}
__host__ __device__ constexpr NibbleLut nibble_lut() {
  return NibbleLut{{nib_word(0, true), nib_word(4, true), nib_word(8, true), nib_word(12, true)},
                   {nib_word(0, false), nib_word(4, false), nib_word(8, false), nib_word(12, false)}};
}

// mask_bucket (kernels.py:125-134): fields >= prefix_len zeroed (decode as A).
__device__ __forceinline__ void mask_words(uint64_t w[4], uint32_t prefix_len) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // fields 32k .. 32k+31 of word k survive below prefix_len
    const int keep = min(max(int(prefix_len) - 32 * k, 0), 32);
    w[k] &= keep == 32 ? ~0ull : ((1ull << (2 * keep)) - 1ull);
  }
}

// Table lookup of four nibble indices (one per byte of idx, each 0..15).
__device__ __forceinline__ uint32_t nib_lookup(uint32_t idx, const uint32_t t[4]) {
  // selector nibbles: byte i's index in bits 4i..4i+2 (PRMT's bit 3 would
  // request sign replication, so only the low three bits are used)
  const uint32_t sel = (idx & 0x7u) | ((idx >> 4) & 0x70u) | ((idx >> 8) & 0x700u) | ((idx >> 12) & 0x7000u);
  const uint32_t a = __byte_perm(t[0], t[1], sel);  // entries 0..7
  const uint32_t b = __byte_perm(t[2], t[3], sel);  // entries 8..15
  const uint32_t hi8 = ((idx >> 3) & 0x01010101u) * 0xFFu;  // bytes whose index is >= 8
  return (a & ~hi8) | (b & hi8);
}

struct NibbleTrace {
  uint64_t masked[4], lo[4], hi[4];
  uint32_t sad[4];
};

// count_bucket_nibble (kernels.py:161-211) on the masked words.
template <bool kTrace>
__device__ __forceinline__ uint32_t nibble_count(const uint64_t m[4], uint32_t prefix_len, uint32_t symbol,
                                                 NibbleTrace* tr) {
  constexpr NibbleLut L = nibble_lut();
  const uint32_t shift = symbol << 1;
  uint32_t sad_total = 0;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t lo32[2], hi32[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t x = uint32_t(m[g] >> (32 * h));
      lo32[h] = nib_lookup(x & 0x0F0F0F0Fu, L.lo);          // phase 1: low nibbles, complemented table
      hi32[h] = nib_lookup((x >> 4) & 0x0F0F0F0Fu, L.hi);   //          high nibbles, plain table
    }
    const uint64_t lo_w = uint64_t(lo32[0]) | (uint64_t(lo32[1]) << 32);
    const uint64_t hi_w = uint64_t(hi32[0]) | (uint64_t(hi32[1]) << 32);
    // phase 2: 64-bit shifts; the fill / mask keeps bits 0..1 of every byte
    const uint64_t slo = (lo_w >> shift) | 0xFCFCFCFCFCFCFCFCull;
    const uint64_t shi = (hi_w >> shift) & 0x0303030303030303ull;
    // phase 3: sum of |lo - hi| over the group's 8 bytes
    const uint32_t sad = __vsadu4(uint32_t(slo), uint32_t(shi)) + __vsadu4(uint32_t(slo >> 32), uint32_t(shi >> 32));
    sad_total += sad;
    if constexpr (kTrace) {
      tr->masked[g] = m[g];
      tr->lo[g] = lo_w;
      tr->hi[g] = hi_w;
      tr->sad[g] = sad;
    }
  }
  const uint32_t raw = 8160u - sad_total;
  return symbol == 0u ? raw - (128u - prefix_len) : raw;
}

__device__ __forceinline__ void load_bucket(const uint8_t* blocks, uint64_t i, uint64_t w[4]) {
  ld256<1>(blocks + i * 32, w[0], w[1], w[2], w[3]);
}

// All four counts (symbols == nullptr) or one symbol's count per query.
// out: 4 x u32 per query (all four) or 1 x u32.  Bad prefix_len / symbol:
// status bit 1, zeros written.
template <int kMethod>
__global__ void __launch_bounds__(256) k_bucket_count(const uint8_t* __restrict__ blocks,
                                                      const uint32_t* __restrict__ prefix_lens,
                                                      const uint8_t* __restrict__ symbols, uint64_t count,
                                                      uint32_t* __restrict__ out, uint32_t* __restrict__ err) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint32_t pl = prefix_lens[i];
    const uint32_t sym = symbols ? symbols[i] : 0u;
    const bool ok = pl <= 128u && sym < 4u;
    if (!ok && err) atomicOr(err, 1u);
    uint64_t w[4];
    load_bucket(blocks, i, w);
    mask_words(w, ok ? pl : 0u);
    const uint32_t p = ok ? pl : 0u;
    if (symbols) {
      uint32_t c;
      if constexpr (kMethod == 0) {
        c = p ? count1<4>(w, p - 1u, sym) : 0u;
      } else {
        c = nibble_count<false>(w, p, sym, nullptr);
      }
      out[i] = ok ? c : 0u;
    } else {
      uint32_t c4[4] = {0u, 0u, 0u, 0u};
      if constexpr (kMethod == 0) {
        if (p) count4<4>(w, p - 1u, c4);
      } else {
#pragma unroll
        for (uint32_t s = 0; s < 4; ++s) c4[s] = nibble_count<false>(w, p, s, nullptr);
      }
      reinterpret_cast<uint4*>(out)[i] = ok ? make_uint4(c4[0], c4[1], c4[2], c4[3]) : make_uint4(0, 0, 0, 0);
    }
  }
}

// mask_bucket for a batch: out = blocks with fields >= prefix_len zeroed.
__global__ void __launch_bounds__(256) k_bucket_mask(const uint8_t* __restrict__ blocks,
                                                     const uint32_t* __restrict__ prefix_lens, uint64_t count,
                                                     uint8_t* __restrict__ out, uint32_t* __restrict__ err) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint32_t pl = prefix_lens[i];
    if (pl > 128u && err) atomicOr(err, 1u);
    uint64_t w[4];
    load_bucket(blocks, i, w);
    mask_words(w, min(pl, 128u));
    ulonglong4* dst = reinterpret_cast<ulonglong4*>(out + i * 32);
    *dst = make_ulonglong4(w[0], w[1], w[2], w[3]);
  }
}

// The nibble pipeline with its trace (kernels.py:101-115): per query 15 u64
// = masked words[4], lookup lo words[4], lookup hi words[4], then
// (group SADs packed 16 bits each), (sad_total | raw_count << 32), count.
__global__ void __launch_bounds__(128) k_bucket_nibble_trace(const uint8_t* __restrict__ blocks,
                                                             const uint32_t* __restrict__ prefix_lens,
                                                             const uint8_t* __restrict__ symbols, uint64_t count,
                                                             uint64_t* __restrict__ trace,
                                                             uint32_t* __restrict__ err) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t pl = prefix_lens[i], sym = symbols[i];
  uint64_t* t = trace + i * 15;
  if (pl > 128u || sym > 3u) {
    if (err) atomicOr(err, 1u);
    for (int q = 0; q < 15; ++q) t[q] = 0;
    return;
  }
  uint64_t w[4];
  load_bucket(blocks, i, w);
  mask_words(w, pl);
  NibbleTrace tr;
  const uint32_t c = nibble_count<true>(w, pl, sym, &tr);
  uint32_t sad_total = 0;
  for (int g = 0; g < 4; ++g) {
    t[g] = tr.masked[g];
    t[4 + g] = tr.lo[g];
    t[8 + g] = tr.hi[g];
    sad_total += tr.sad[g];
  }
  t[12] = uint64_t(tr.sad[0]) | (uint64_t(tr.sad[1]) << 16) | (uint64_t(tr.sad[2]) << 32) |
          (uint64_t(tr.sad[3]) << 48);
  t[13] = uint64_t(sad_total) | (uint64_t(8160u - sad_total) << 32);
  t[14] = c;
}

}  // namespace fmg
