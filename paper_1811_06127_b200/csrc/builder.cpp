// Native FM-index builder: suffix array by induced sorting (SA-IS), BWT,
// 128-character occurrence buckets and sampled suffix-array entries.
//
// Replaces the reference's offline construction path, which is pure Python
// and does not scale past ~16 Mbp:
//   suffix.py:21-46  build_suffix_array (prefix doubling, tuple keys)
//   suffix.py:49-71  bwt_from_sa        ('$' at sentinel_row)
//   index.py:57-64   build_c_table      (c[4] == n, '$' not counted)
//   index.py:67-101  build_index        ('$' packed as code 0, bases are
//                                        exclusive running counts of the raw
//                                        packed transform, zero padding)
// The suffix array of text+'$' is unique, so any correct construction yields
// the same transform, bases and samples; the .fmi written from these arrays
// is byte-identical to serialize_index(build_index(text)) (pinned by
// tests/test_builder.py against fixtures made with the reference itself).
//
// Host code only (no CUDA); compiled into libfmgpu.so next to the kernels.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fmgpu_internal.h"

namespace {

// ---------------------------------------------------------------------------
// SA-IS (induced sorting).  `s` has length n, s[n-1] is the unique smallest
// symbol (the sentinel), all symbols lie in [0, K).  Idx must hold n.
// ---------------------------------------------------------------------------

class TypeBits {
 public:
  explicit TypeBits(size_t n) : w_((n + 63) / 64, 0) {}
  inline void set_s(size_t i) { w_[i >> 6] |= (1ull << (i & 63)); }
  inline bool is_s(size_t i) const { return (w_[i >> 6] >> (i & 63)) & 1ull; }

 private:
  std::vector<uint64_t> w_;
};

template <typename Idx>
inline bool is_lms(const TypeBits& t, Idx i) {
  return i > 0 && t.is_s(i) && !t.is_s(i - 1);
}

template <typename Char, typename Idx>
void bucket_bounds(const Char* s, Idx n, Idx K, std::vector<Idx>& bkt, bool ends) {
  std::fill(bkt.begin(), bkt.end(), Idx(0));
  for (Idx i = 0; i < n; ++i) bkt[s[i]]++;
  Idx sum = 0;
  for (Idx c = 0; c < K; ++c) {
    sum += bkt[c];
    bkt[c] = ends ? sum : sum - bkt[c];
  }
}

template <typename Char, typename Idx>
void induce(const Char* s, Idx* SA, Idx n, Idx K, const TypeBits& t, std::vector<Idx>& bkt) {
  const Idx EMPTY = ~Idx(0);
  // L-type suffixes, left to right, from bucket heads.
  bucket_bounds(s, n, K, bkt, false);
  for (Idx i = 0; i < n; ++i) {
    Idx j = SA[i];
    if (j != EMPTY && j > 0 && !t.is_s(j - 1)) SA[bkt[s[j - 1]]++] = j - 1;
  }
  // S-type suffixes, right to left, from bucket tails.
  bucket_bounds(s, n, K, bkt, true);
  for (Idx i = n; i-- > 0;) {
    Idx j = SA[i];
    if (j != EMPTY && j > 0 && t.is_s(j - 1)) SA[--bkt[s[j - 1]]] = j - 1;
  }
}

template <typename Char, typename Idx>
void sais(const Char* s, Idx* SA, Idx n, Idx K) {
  const Idx EMPTY = ~Idx(0);
  if (n == 1) {
    SA[0] = 0;
    return;
  }
  TypeBits t(n);
  t.set_s(n - 1);
  for (Idx i = n - 1; i-- > 0;) {
    if (s[i] < s[i + 1] || (s[i] == s[i + 1] && t.is_s(i + 1))) t.set_s(i);
  }
  std::vector<Idx> bkt(K);

  // Stage 1: sort LMS substrings by one round of induced sorting.
  std::fill(SA, SA + n, EMPTY);
  bucket_bounds(s, n, K, bkt, true);
  for (Idx i = 1; i < n; ++i)
    if (is_lms(t, i)) SA[--bkt[s[i]]] = i;
  induce(s, SA, n, K, t, bkt);

  // Compact the sorted LMS positions into SA[0, n1).
  Idx n1 = 0;
  for (Idx i = 0; i < n; ++i)
    if (is_lms(t, SA[i])) SA[n1++] = SA[i];

  // Name LMS substrings; names land in SA[n1 + pos/2] (distinct slots since
  // LMS positions are at least two apart).
  std::fill(SA + n1, SA + n, EMPTY);
  Idx name = 0, prev = EMPTY;
  for (Idx i = 0; i < n1; ++i) {
    Idx pos = SA[i];
    bool diff = false;
    for (Idx d = 0; d < n; ++d) {
      if (prev == EMPTY || s[pos + d] != s[prev + d] || t.is_s(pos + d) != t.is_s(prev + d)) {
        diff = true;
        break;
      }
      if (d > 0 && (is_lms(t, pos + d) || is_lms(t, prev + d))) break;
    }
    if (diff) {
      ++name;
      prev = pos;
    }
    SA[n1 + pos / 2] = name - 1;
  }
  // Reduced string: names in text order.
  std::vector<Idx> s1(n1);
  {
    Idx j = 0;
    for (Idx i = n1; i < n; ++i)
      if (SA[i] != EMPTY) s1[j++] = SA[i];
  }

  // Stage 2: sort the reduced problem (recursively when names repeat).
  std::vector<Idx> sa1(n1);
  if (name < n1) {
    sais<Idx, Idx>(s1.data(), sa1.data(), n1, name);
  } else {
    for (Idx i = 0; i < n1; ++i) sa1[s1[i]] = i;
  }

  // Stage 3: induce the full order from the sorted LMS suffixes.
  {
    Idx j = 0;
    for (Idx i = 1; i < n; ++i)
      if (is_lms(t, i)) s1[j++] = i;  // s1 now maps reduced index -> text position
  }
  for (Idx i = 0; i < n1; ++i) sa1[i] = s1[sa1[i]];
  std::fill(SA, SA + n, EMPTY);
  bucket_bounds(s, n, K, bkt, true);
  for (Idx i = n1; i-- > 0;) {
    Idx j = sa1[i];
    SA[--bkt[s[j]]] = j;
  }
  induce(s, SA, n, K, t, bkt);
}

inline void check_codes(const uint8_t* codes, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (codes[i] > 3) throw std::invalid_argument("symbol code outside [0, 4)");
}

// Suffix array of codes + '$' (length n+1), '$' ranking below every symbol.
void suffix_array_u32(const uint8_t* codes, uint64_t n, uint32_t* sa) {
  std::vector<uint8_t> s(n + 1);
  for (uint64_t i = 0; i < n; ++i) s[i] = uint8_t(codes[i] + 1);
  s[n] = 0;
  sais<uint8_t, uint32_t>(s.data(), sa, uint32_t(n + 1), 5u);
}

template <typename F>
void parallel_for(uint64_t count, int nthreads, F&& fn) {
  if (nthreads <= 1 || count < (1u << 16)) {
    fn(uint64_t(0), count);
    return;
  }
  std::vector<std::thread> pool;
  uint64_t chunk = (count + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    uint64_t lo = std::min(count, chunk * t), hi = std::min(count, chunk * (t + 1));
    if (lo < hi) pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int fmb_suffix_array(const uint8_t* codes, uint64_t n, uint32_t* sa_out) {
  return fmg::guard([&] {
    if (n == 0) throw std::invalid_argument("reference is empty");
    if (n + 1 >= 0xFFFFFFFFull) throw std::invalid_argument("reference too long for 32-bit rows");
    check_codes(codes, n);
    suffix_array_u32(codes, n, sa_out);
  });
}

// Builds every array the .fmi format stores (serialize.py:82-104):
//   bucket_records: ceil((n+1)/128) records of 64 bytes = 4 x u64 LE base +
//                   32 bytes packed chars (alphabet.py:53-56 bit order);
//   sa_samples:     sa[0], sa[32], ... (n/32 + 1 entries, index.py:93);
//   c[5], sentinel_row.
int fmb_build(const uint8_t* codes, uint64_t n, uint8_t* bucket_records, uint64_t* sa_samples,
              uint64_t* c_out, uint64_t* sentinel_row_out, int nthreads) {
  return fmg::guard([&] {
    if (n == 0) throw std::invalid_argument("reference is empty");
    if (n + 1 >= 0xFFFFFFFFull) throw std::invalid_argument("reference too long for 32-bit rows");
    check_codes(codes, n);
    const uint64_t rows = n + 1;
    std::vector<uint32_t> sa(rows);
    suffix_array_u32(codes, n, sa.data());

    // BWT codes with '$' stored as 0 (index.py:83); locate the sentinel row.
    std::vector<uint8_t> bwt(rows);
    uint64_t sentinel_row = ~0ull;
    for (uint64_t i = 0; i < rows; ++i) {
      uint32_t p = sa[i];
      if (p == 0) {
        sentinel_row = i;
        bwt[i] = 0;
      } else {
        bwt[i] = codes[p - 1];
      }
    }
    if (sentinel_row == ~0ull) throw std::runtime_error("suffix array holds no entry for position 0");

    const uint64_t nb = (rows + 127) / 128;
    // Per-bucket raw counts (with '$' in the A lane) and packed chars.
    std::vector<uint64_t> counts(nb * 4, 0);
    parallel_for(nb, nthreads, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t b = lo; b < hi; ++b) {
        uint8_t* rec = bucket_records + b * 64;
        uint8_t* chars = rec + 32;
        std::memset(chars, 0, 32);
        uint64_t cnt[4] = {0, 0, 0, 0};
        uint64_t start = b * 128, end = std::min(rows, start + 128);
        for (uint64_t i = start; i < end; ++i) {
          uint64_t r = i - start;
          uint8_t code = bwt[i];
          chars[r >> 2] |= uint8_t(code << ((r & 3) << 1));
          cnt[code]++;
        }
        for (int s = 0; s < 4; ++s) counts[b * 4 + s] = cnt[s];
      }
    });
    uint64_t base[4] = {0, 0, 0, 0};
    for (uint64_t b = 0; b < nb; ++b) {
      uint8_t* rec = bucket_records + b * 64;
      std::memcpy(rec, base, 32);  // little-endian host
      for (int s = 0; s < 4; ++s) base[s] += counts[b * 4 + s];
    }
    // C table over the transform without '$' (index.py:78-81).
    uint64_t totals[4] = {base[0] - 1, base[1], base[2], base[3]};
    c_out[0] = 0;
    for (int s = 0; s < 4; ++s) c_out[s + 1] = c_out[s] + totals[s];
    for (uint64_t i = 0, j = 0; i < rows; i += 32, ++j) sa_samples[j] = sa[i];
    *sentinel_row_out = sentinel_row;
  });
}

}  // extern "C"
