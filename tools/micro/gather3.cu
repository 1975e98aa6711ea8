// Does a 128-byte line read by 4 lanes in ONE instruction cost one DRAM
// request?  Compares random 32 B reads (1 lane), 64 B (2 lanes) and 128 B
// (4 lanes) per access, same number of accesses.
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>
#include <cuda_runtime.h>

template <int LANES>
__global__ void g(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ idx, uint64_t count,
                  unsigned long long* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t a = t / LANES;
  const int q = t % LANES;
  if (a >= count) return;
  const uint8_t* p = buf + (uint64_t)idx[a] * (32 * LANES) + 32 * q;
  uint64_t a0, a1, a2, a3;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p));
  if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345) atomicAdd(sink, 1ull);
}

template <int LANES>
void run(const uint8_t* buf, uint64_t total, unsigned long long* sink, uint64_t count) {
  std::vector<uint32_t> h(count);
  std::mt19937_64 rng(LANES);
  for (auto& x : h) x = uint32_t(rng() % (total / (32 * LANES)));
  uint32_t* d; cudaMalloc(&d, count * 4); cudaMemcpy(d, h.data(), count * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint64_t threads = count * LANES;
  g<LANES><<<threads / 256, 256>>>(buf, d, count, sink);
  cudaEventRecord(e0);
  g<LANES><<<threads / 256, 256>>>(buf, d, count, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%3d B/access (%d lanes): %.1f us, %.1f G accesses/s, %.1f GB/s useful\n", 32 * LANES, LANES, ms * 1e3,
         count / ms / 1e6, count * 32.0 * LANES / ms / 1e6);
  cudaFree(d);
}

int main() {
  const uint64_t total = 4ull << 30, count = 1ull << 25;
  uint8_t* buf; unsigned long long* sink;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total); cudaMalloc(&sink, 8);
  run<1>(buf, total, sink, count);
  run<2>(buf, total, sink, count);
  run<4>(buf, total, sink, count);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
