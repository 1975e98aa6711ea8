// GPU index construction: suffix array by prefix doubling on the device,
// then BWT, bucket records and samples, all in HBM.
//
// Same outputs as the host SA-IS builder (builder.cpp) and therefore as the
// reference's build_index (suffix.py:21-71, index.py:67-101): the suffix
// array of text+'$' is unique, so any correct construction gives the same
// transform, bases and samples (tests/test_gpu_builder.py checks the two
// builders against each other and the .fmi bytes against the reference's).
//
// Doubling: the first key packs 21 characters of 3 bits ('$' = 0 below
// A..T = 1..4, zero past the end), so suffixes shorter than 21 characters
// compare correctly.  Each round sorts (rank[i], rank[i+h] + 1) 64-bit keys
// with CUB's radix sort (library sort; the index build is off the hot path)
// and re-ranks by group heads; random-like genomes finish after 1-3 rounds.
// Memory: ~36 bytes per character (keys and values double-buffered).

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "fmgpu_internal.h"

namespace {

#define BG_CK(expr)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::fmg::CudaError(std::string(#expr) + " failed: " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) {
    if (n) BG_CK(cudaMalloc(&p, n * sizeof(T)));
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

inline unsigned grid(uint64_t n, unsigned t = 256) { return unsigned((n + t - 1) / t); }

__global__ void k_check_codes(const uint8_t* codes, uint64_t n, uint32_t* bad) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && codes[i] > 3) atomicOr(bad, 1u);
}

// key[i] = 21 chars from i, 3 bits each, '$' (and past the end) = 0.
__global__ void k_initial_keys(const uint8_t* codes, uint64_t n, uint64_t* keys, uint32_t* idx) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > n) return;
  uint64_t k = 0;
#pragma unroll
  for (int j = 0; j < 21; ++j) {
    const uint64_t p = i + j;
    const uint64_t c = p < n ? uint64_t(codes[p]) + 1 : 0;
    k = (k << 3) | c;
  }
  keys[i] = k;
  idx[i] = uint32_t(i);
}

__global__ void k_head_flags(const uint64_t* keys, uint64_t rows, uint32_t* head) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  head[j] = (j == 0 || keys[j] != keys[j - 1]) ? uint32_t(j) : 0u;
}

__global__ void k_flag_count(const uint64_t* keys, uint64_t rows, uint32_t* flags) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  flags[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1u : 0u;
}

// rank[sa[j]] = head[j] (group head = number of suffixes strictly smaller).
__global__ void k_scatter_rank(const uint32_t* sa, const uint32_t* head, uint64_t rows, uint32_t* rank) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < rows) rank[sa[j]] = head[j];
}

__global__ void k_double_keys(const uint32_t* rank, uint64_t rows, uint64_t h, uint64_t* keys, uint32_t* idx) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const uint64_t second = (i + h < rows) ? uint64_t(rank[i + h]) + 1 : 0;
  keys[i] = (uint64_t(rank[i]) << 32) | second;
  idx[i] = uint32_t(i);
}

// BWT code per row ('$' stored as 0, index.py:83) and the sentinel row.
__global__ void k_bwt(const uint32_t* sa, const uint8_t* codes, uint64_t rows, uint8_t* bwt,
                      unsigned long long* sentinel) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  const uint32_t p = sa[j];
  if (p == 0) {
    bwt[j] = 0;
    *sentinel = j;
  } else {
    bwt[j] = codes[p - 1];
  }
}

// Per bucket: packed chars into the record and raw symbol counts.
__global__ void k_bucket_chars(const uint8_t* bwt, uint64_t rows, uint64_t nb, uint8_t* rec, ulonglong4* counts) {
  const uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  uint64_t cnt[4] = {0, 0, 0, 0};
  uint8_t* chars = rec + b * 64 + 32;
  for (int q = 0; q < 32; ++q) {
    uint8_t byte = 0;
    for (int f = 0; f < 4; ++f) {
      const uint64_t i = b * 128 + q * 4 + f;
      if (i < rows) {
        const uint8_t c = bwt[i];
        byte |= uint8_t(c << (2 * f));
        cnt[c]++;
      }
    }
    chars[q] = byte;
  }
  counts[b] = make_ulonglong4(cnt[0], cnt[1], cnt[2], cnt[3]);
}

struct Add4 {
  __device__ __forceinline__ ulonglong4 operator()(const ulonglong4& a, const ulonglong4& b) const {
    return make_ulonglong4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
};

__global__ void k_bucket_bases(const ulonglong4* excl, uint64_t nb, uint8_t* rec) {
  const uint64_t b = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const ulonglong4 v = excl[b];
  uint64_t* base = reinterpret_cast<uint64_t*>(rec + b * 64);
  base[0] = v.x;
  base[1] = v.y;
  base[2] = v.z;
  base[3] = v.w;
}

__global__ void k_samples(const uint32_t* sa, uint64_t count, uint64_t* out) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < count) out[j] = sa[j * 32];
}

}  // namespace

extern "C" int fmb_build_gpu(int device, const uint8_t* codes_host, uint64_t n, uint8_t* bucket_records,
                             uint64_t* sa_samples, uint64_t* c_out, uint64_t* sentinel_row_out,
                             uint32_t* sa_out) {
  return fmg::guard([&] {
    if (n == 0) throw std::invalid_argument("reference is empty");
    if (n + 1 >= 0xFFFFFFFFull) throw std::invalid_argument("reference too long for 32-bit rows");
    int prev = -1;
    BG_CK(cudaGetDevice(&prev));
    BG_CK(cudaSetDevice(device));
    struct Restore {
      int d;
      ~Restore() {
        if (d >= 0) cudaSetDevice(d);
      }
    } restore{prev};
    const uint64_t rows = n + 1;
    Dev<uint8_t> codes(n);
    BG_CK(cudaMemcpy(codes.p, codes_host, n, cudaMemcpyHostToDevice));
    Dev<uint32_t> flag(1);
    BG_CK(cudaMemset(flag.p, 0, 4));
    k_check_codes<<<grid(n), 256>>>(codes.p, n, flag.p);
    uint32_t bad = 0;
    BG_CK(cudaMemcpy(&bad, flag.p, 4, cudaMemcpyDeviceToHost));
    if (bad) throw std::invalid_argument("symbol code outside [0, 4)");

    Dev<uint64_t> keys_a(rows), keys_b(rows);
    Dev<uint32_t> vals_a(rows), vals_b(rows);
    Dev<uint32_t> rank(rows), head(rows);
    // temp storage for the largest CUB call (sort dominates)
    size_t sort_bytes = 0, scan_bytes = 0, red_bytes = 0;
    {
      cub::DoubleBuffer<uint64_t> k(keys_a.p, keys_b.p);
      cub::DoubleBuffer<uint32_t> v(vals_a.p, vals_b.p);
      BG_CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, k, v, rows));
      BG_CK(cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, head.p, head.p, cub::Max(), rows));
      BG_CK(cub::DeviceReduce::Sum(nullptr, red_bytes, head.p, flag.p, rows));
    }
    Dev<uint8_t> tmp(std::max(sort_bytes, std::max(scan_bytes, red_bytes)));
    const size_t tmp_bytes = std::max(sort_bytes, std::max(scan_bytes, red_bytes));

    k_initial_keys<<<grid(rows), 256>>>(codes.p, n, keys_a.p, vals_a.p);
    BG_CK(cudaGetLastError());
    uint64_t h = 21;
    int end_bit = 63;
    uint32_t* sa = nullptr;
    for (int round = 0;; ++round) {
      if (round > 40) throw std::runtime_error("prefix doubling did not converge");
      cub::DoubleBuffer<uint64_t> k(keys_a.p, keys_b.p);
      cub::DoubleBuffer<uint32_t> v(vals_a.p, vals_b.p);
      size_t tb = tmp_bytes;
      BG_CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k, v, rows, 0, end_bit));
      sa = v.Current();
      const uint64_t* sorted = k.Current();
      // unique count
      k_flag_count<<<grid(rows), 256>>>(sorted, rows, head.p);
      tb = tmp_bytes;
      BG_CK(cub::DeviceReduce::Sum(tmp.p, tb, head.p, flag.p, rows));
      uint32_t distinct = 0;
      BG_CK(cudaMemcpy(&distinct, flag.p, 4, cudaMemcpyDeviceToHost));
      if (uint64_t(distinct) == rows) break;
      // rank = group head position
      k_head_flags<<<grid(rows), 256>>>(sorted, rows, head.p);
      tb = tmp_bytes;
      BG_CK(cub::DeviceScan::InclusiveScan(tmp.p, tb, head.p, head.p, cub::Max(), rows));
      k_scatter_rank<<<grid(rows), 256>>>(sa, head.p, rows, rank.p);
      // next keys: (rank[i], rank[i+h] + 1), into the buffers not holding sa
      uint64_t* nk = (k.Current() == keys_a.p) ? keys_b.p : keys_a.p;
      uint32_t* nv = (sa == vals_a.p) ? vals_b.p : vals_a.p;
      k_double_keys<<<grid(rows), 256>>>(rank.p, rows, h, nk, nv);
      BG_CK(cudaGetLastError());
      // make the next round's DoubleBuffer start from nk / nv
      if (nk != keys_a.p) std::swap(keys_a.p, keys_b.p);
      if (nv != vals_a.p) std::swap(vals_a.p, vals_b.p);
      int bits = 1;
      while ((uint64_t(1) << bits) <= rows + 1) ++bits;
      end_bit = 32 + bits;
      h *= 2;
    }
    if (sa_out) BG_CK(cudaMemcpy(sa_out, sa, rows * 4, cudaMemcpyDeviceToHost));

    // BWT, buckets, C table, samples
    Dev<uint8_t> bwt(rows);
    Dev<unsigned long long> sent(1);
    k_bwt<<<grid(rows), 256>>>(sa, codes.p, rows, bwt.p, sent.p);
    const uint64_t nb = (rows + 127) / 128;
    Dev<uint8_t> rec(nb * 64);
    Dev<ulonglong4> counts(nb), excl(nb);
    k_bucket_chars<<<grid(nb), 256>>>(bwt.p, rows, nb, rec.p, counts.p);
    size_t sb = 0;
    BG_CK(cub::DeviceScan::ExclusiveScan(nullptr, sb, counts.p, excl.p, Add4(), make_ulonglong4(0, 0, 0, 0), nb));
    Dev<uint8_t> stmp(sb);
    BG_CK(cub::DeviceScan::ExclusiveScan(stmp.p, sb, counts.p, excl.p, Add4(), make_ulonglong4(0, 0, 0, 0), nb));
    k_bucket_bases<<<grid(nb), 256>>>(excl.p, nb, rec.p);
    const uint64_t ns = n / 32 + 1;
    Dev<uint64_t> samp(ns);
    k_samples<<<grid(ns), 256>>>(sa, ns, samp.p);
    BG_CK(cudaGetLastError());
    BG_CK(cudaMemcpy(bucket_records, rec.p, nb * 64, cudaMemcpyDeviceToHost));
    BG_CK(cudaMemcpy(sa_samples, samp.p, ns * 8, cudaMemcpyDeviceToHost));
    unsigned long long sentinel = 0;
    BG_CK(cudaMemcpy(&sentinel, sent.p, 8, cudaMemcpyDeviceToHost));
    ulonglong4 last_excl, last_cnt;
    BG_CK(cudaMemcpy(&last_excl, excl.p + nb - 1, sizeof(ulonglong4), cudaMemcpyDeviceToHost));
    BG_CK(cudaMemcpy(&last_cnt, counts.p + nb - 1, sizeof(ulonglong4), cudaMemcpyDeviceToHost));
    const uint64_t tot[4] = {last_excl.x + last_cnt.x - 1, last_excl.y + last_cnt.y, last_excl.z + last_cnt.z,
                             last_excl.w + last_cnt.w};
    c_out[0] = 0;
    for (int s = 0; s < 4; ++s) c_out[s + 1] = c_out[s] + tot[s];
    *sentinel_row_out = sentinel;
  });
}
