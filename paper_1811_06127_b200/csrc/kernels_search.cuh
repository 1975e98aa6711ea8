// Exact backward search and position recovery kernels (search.py:74-94, 172-208).
// Part of libfmgpu.so (sm_100a); included once by fmgpu.cu.
#pragma once

#include <cstdint>

#include "occ_device.cuh"

namespace fmg {

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
// k-mer table: lut[x] = the interval exact_search returns for the K-mer x
// (character t of x in bits 2t), including the first empty interval where
// that search stopped.  A pattern of length m >= K starts from the entry of
// its last K characters at position m-1-K, skipping K dependent steps — the
// result is identical because the entry IS what those K steps produce.
// pp.words == nullptr makes k_exact search the K-mers x = 0 .. count-1
// themselves (how the table is built).

// Prefix interval table: level j (1 <= j <= k) holds the interval of every
// string x of length j, key(x) = sum x_t 4^t (x_0 = first character), at
// base[off(j) + key]; absent strings hold some k > l.  Prepending b to S
// gives key(bS) = b + 4 key(S), so the four children of a node whose string
// S is shorter than k sit in ONE aligned 32-byte sector of level |S| + 1.
struct PrefixTable {
  const uint2* base = nullptr;
  uint32_t k = 0;
  __host__ __device__ static uint32_t off(uint32_t j) { return ((1u << (2 * j)) - 4u) / 3u; }  // j <= 15
  static uint64_t off64(uint32_t j) { return ((uint64_t(1) << (2 * j)) - 4u) / 3u; }
};

#ifndef FMG_EXACT_PRED_LOW
#define FMG_EXACT_PRED_LOW 1  // k_exact (W = 2): predicated low-line load instead of a branch
#endif

struct KmerTable {
  const uint2* lut = nullptr;
  uint32_t k = 0;
  const uint2* pbase = nullptr;  // the prefix table (levels 1..pk) for patterns shorter than k
  uint32_t pk = 0;
};

template <bool kPacked, int W>
__global__ void __launch_bounds__(256) k_exact(IndexView ix, PackedPatterns pp, CodePatterns cp, uint64_t count,
                                               uint2* __restrict__ out, unsigned long long* __restrict__ steps,
                                               KmerTable kt) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t work = 0;  // work_unit per step
  uint64_t pat = 0;          // packed form
  const uint8_t* codes = nullptr;  // general form
  int i = -1;
  uint32_t k = 1, l = 0;
  auto start = [&](uint64_t qq) {
    uint32_t m, b;
    if (kPacked) {
      pat = pp.words ? pp.words[qq] : qq;
      m = pp.m;
      b = uint32_t(pat >> (2 * (m - 1))) & 3u;
    } else {
      const uint64_t o0 = cp.offsets[qq], o1 = cp.offsets[qq + 1];
      codes = cp.codes + o0;
      m = uint32_t(o1 - o0);
      b = codes[m - 1];
    }
    // start after the last d characters, d = K (level-K table) or, for a
    // shorter pattern, min(m, prefix depth) from the prefix table's level d
    const bool full = kt.lut && m >= kt.k;
    const uint32_t d = full ? kt.k : (kt.pbase ? min(m, kt.pk) : 0u);
    if (d > 0) {
      uint32_t key = 0;
      if (kPacked) {
        key = uint32_t((pat >> (2 * (m - d))) & ((uint64_t(1) << (2 * d)) - 1u));  // d <= 16
      } else {
        for (uint32_t t = 0; t < d; ++t) key |= uint32_t(__ldg(codes + m - d + t) & 3u) << (2 * t);
      }
      const uint2 e = __ldg(full ? kt.lut + key : kt.pbase + PrefixTable::off(d) + key);
      work += 1u;  // one random table gather: counted as a fetched line, not as an Occ step
      k = e.x;
      l = e.y;
      i = int(m) - 1 - int(d);
      return;
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
    // (Loading the low line unconditionally, to drop the branch, costs a
    // second memory request when both ends share a line: config 4 12.0 ->
    // 9.0 G seeds/s.  W = 2 uses a predicated load instead: no request,
    // no branch.)
    if constexpr (W == 2 && FMG_EXACT_PRED_LOW) {
      uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      ld256_pred(jl != jh, ix.lines + size_t(jl) * LineTraits<2>::kBytes, a0, a1, a2, a3);
      const bool same = jl == jh;
      bl[0] = same ? bh[0] : uint32_t(a0);
      bl[1] = same ? bh[1] : uint32_t(a0 >> 32);
      bl[2] = same ? bh[2] : uint32_t(a1);
      bl[3] = same ? bh[3] : uint32_t(a1 >> 32);
      wl[0] = same ? wh[0] : a2;
      wl[1] = same ? wh[1] : a3;
      ol = occ1_from_line<W>(ix, bl, wl, low, rl, sym);
    } else if (jl != jh) {
      load_line<W, false>(ix, jl, rl, bl, wl);
      ol = occ1_from_line<W>(ix, bl, wl, low, rl, sym);
    } else {
      ol = occ1_from_line<W>(ix, bh, wh, low, rl, sym);
    }
    const uint32_t oh = occ1_from_line<W>(ix, bh, wh, l, rh, sym);
    const uint32_t cs = c_of(ix, sym);
    k = cs + ol + 1u;
    l = cs + oh;
    work += work_unit(jl != jh ? 2u : 1u);
  }
  flush_work(steps, work);
}


// Level j of the k-mer / prefix interval table from level j-1 (`parent`,
// null for j = 1): entry x (x_0 = first character in bits 0..1) is the
// interval exact_search returns for x — extend_backward of the entry of
// x[1..] = x >> 2 by x_0, or that entry unchanged when it is already the
// first empty interval (search.py:88-93).  One Occ step per entry; the four
// siblings share their parent's lines (L1 hits).
template <int W>
__global__ void __launch_bounds__(256) k_lut_level(IndexView ix, const uint2* __restrict__ parent,
                                                   uint2* __restrict__ out, uint64_t cnt) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  const uint32_t sym = uint32_t(q & 3u);
  const uint32_t cs = c_of(ix, sym);
  if (parent == nullptr) {  // init_interval, search.py:50-57
    out[q] = make_uint2(cs + 1u, c_of(ix, sym + 1u));
    return;
  }
  const uint2 e = parent[q >> 2];
  if (e.x > e.y) {
    out[q] = e;
    return;
  }
  constexpr uint32_t kC = LineTraits<W>::kChars;
  const uint32_t low = e.x - 1u, l = e.y;  // e.x >= 1 on every non-empty interval
  const uint32_t jh = line_of<W>(l), jl = line_of<W>(low);
  uint32_t bh[4], bl[4];
  uint64_t wh[W], wl[W];
  load_line<W, 0>(ix, jh, l - jh * kC, bh, wh);
  load_line<W, 0>(ix, jl, low - jl * kC, bl, wl);
  out[q] = make_uint2(cs + occ1_from_line<W>(ix, bl, wl, low, low - jl * kC, sym) + 1u,
                      cs + occ1_from_line<W>(ix, bh, wh, l, l - jh * kC, sym));
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

// reconstruct_reference (search.py:270-286) in parallel.  The predecessor
// cycle from row 0 (suffix n) to the sentinel row (suffix 0) visits every row
// once; the sampled rows (row % 32 == 0, index.py:93) cut it into segments of
// ~32 steps.  Segment j starts at row 32j, whose text position samples[j] is
// known, and writes text[pos - 1], text[pos - 2], ... until it reaches the
// next sampled row or the sentinel row, so every text position is written
// exactly once.  Bit 2 of err: the walk left [0, n] (corrupt index).
template <int W>
__global__ void __launch_bounds__(256) k_reconstruct(IndexView ix, uint64_t n_samples, uint8_t* __restrict__ text,
                                                     uint32_t* __restrict__ err) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n_samples; j += stride) {
    uint32_t row = uint32_t(j) << 5, pos = ix.samples[j];
    for (uint32_t steps = 0; row != ix.sentinel_row; ++steps) {
      if (pos == 0u || pos > ix.n || steps > 64u * 1024u * 1024u) {
        if (err) atomicOr(err, 2u);
        break;
      }
      uint32_t sym;
      const uint32_t prev = psi_step<W>(ix, row, sym);
      text[pos - 1u] = uint8_t(sym);
      --pos;
      row = prev;
      if ((row & 31u) == 0u) break;
    }
  }
}

template <int W>
__global__ void k_psi(IndexView ix, const uint32_t* __restrict__ rows, uint64_t count, uint8_t* __restrict__ out_sym,
                      uint32_t* __restrict__ out_row, uint32_t* __restrict__ err) {
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const uint32_t row = rows[q];
  if (row > ix.n) {
    if (err) atomicOr(err, 1u);
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
      if (err) atomicOr(err, 1u);
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
        if (err) atomicOr(err, 2u);
        out_pos[q] = 0xFFFFFFFFu;
        break;
      }
    }
  }
}

}  // namespace fmg
