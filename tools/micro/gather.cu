// Random-gather microbenchmark: time and DRAM bytes per random access of
// 32/64/128 B from a 4 GiB buffer.  Offsets are precomputed (uniform random,
// aligned) so the kernel is pure loads; U independent accesses per thread.
// Used to choose the index layout.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int BYTES, int U>
__global__ void gather(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ idx, uint64_t count,
                       unsigned long long* sink) {
  uint64_t base = (blockIdx.x * (uint64_t)blockDim.x) * U + threadIdx.x;
  uint64_t acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint64_t i = base + (uint64_t)u * blockDim.x;
    if (i >= count) break;
    const uint8_t* p = buf + (uint64_t)idx[i] * BYTES;
#pragma unroll
    for (int o = 0; o < BYTES; o += 32) {
      uint64_t a0, a1, a2, a3;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p + o));
      acc ^= a0 ^ a1 ^ a2 ^ a3;
    }
  }
  if (acc == 0x12345) atomicAdd(sink, 1ull);
}

template <int BYTES, int U>
void run(const uint8_t* buf, uint64_t total, const uint32_t* d_idx_all, unsigned long long* sink, uint64_t count) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const unsigned blocks = unsigned((count + 256 * U - 1) / (256 * U));
  const uint32_t* d_idx = d_idx_all + (BYTES == 32 ? 0 : BYTES == 64 ? 1 : 2) * count;
  for (int w = 0; w < 2; ++w) gather<BYTES, U><<<blocks, 256>>>(buf, d_idx, count, sink);
  cudaEventRecord(e0);
  gather<BYTES, U><<<blocks, 256>>>(buf, d_idx, count, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%3d B/access U=%d: %.1f us, %.1f G accesses/s, useful %.1f GB/s\n", BYTES, U, ms * 1e3,
         count / ms / 1e6, count * (double)BYTES / ms / 1e6);
}

int main() {
  const uint64_t total = 4ull << 30, count = 1ull << 25;
  uint8_t* buf; unsigned long long* sink; uint32_t* d_idx;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  cudaMalloc(&sink, 8);
  std::vector<uint32_t> h(3 * count);
  std::mt19937_64 rng(1);
  for (int k = 0; k < 3; ++k) {
    uint64_t nchunks = total / (32u << k);
    for (uint64_t i = 0; i < count; ++i) h[k * count + i] = uint32_t(rng() % nchunks);
  }
  cudaMalloc(&d_idx, h.size() * 4);
  cudaMemcpy(d_idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  run<32, 1>(buf, total, d_idx, sink, count);
  run<32, 4>(buf, total, d_idx, sink, count);
  run<64, 1>(buf, total, d_idx, sink, count);
  run<64, 4>(buf, total, d_idx, sink, count);
  run<128, 1>(buf, total, d_idx, sink, count);
  run<128, 4>(buf, total, d_idx, sink, count);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
