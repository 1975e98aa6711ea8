// Dependent-load latency on B200: one thread chases a random cyclic
// permutation of 32-byte slots in a buffer of the given size (the access
// pattern of one exact-search chain), timed with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/chase tools/micro/chase.cu
//   ./tools/micro/chase
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void chase(const uint64_t* __restrict__ buf, uint64_t start, int hops, int nc, unsigned long long* out) {
  uint64_t p = start;
  const long long t0 = clock64();
  for (int h = 0; h < hops; ++h) {
    uint64_t v, a1 = 0, a2 = 0, a3 = 0;
    if (nc == 1) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(buf + p * 4));
    else if (nc == 0) asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(buf + p * 4));
    else if (nc == 2) asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(v), "=l"(a1) : "l"(buf + p * 4));
    else asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(buf + p * 4));
    p = v + ((a1 ^ a2 ^ a3) & 0);
  }
  const long long t1 = clock64();
  out[0] = (unsigned long long)(t1 - t0);
  out[1] = p;
}

int main() {
  const size_t sizes[] = {size_t(512) << 10, size_t(8) << 20, size_t(64) << 20, size_t(1) << 30};
  for (size_t bytes : sizes) {
    const uint64_t slots = bytes / 32;
    std::vector<uint64_t> perm(slots);
    for (uint64_t i = 0; i < slots; ++i) perm[i] = i;
    std::mt19937_64 rng(7);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<uint64_t> host(slots * 4, 0);
    for (uint64_t i = 0; i < slots; ++i) host[perm[i] * 4] = perm[(i + 1) % slots];  // one random cycle
    uint64_t* d = nullptr;
    unsigned long long* o = nullptr;
    cudaMalloc(&d, bytes);
    cudaMalloc(&o, 16);
    cudaMemcpy(d, host.data(), bytes, cudaMemcpyHostToDevice);
    for (int nc = 0; nc < 4; ++nc) {
      const int hops = 20000;
      chase<<<1, 1>>>(d, perm[0], hops, nc, o);  // warm (L2 for small buffers)
      chase<<<1, 1>>>(d, perm[0], hops, nc, o);
      unsigned long long r[2];
      cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("buffer %8zu KB  %s  %.0f cycles per dependent load\n", bytes >> 10, nc == 0 ? "ld.global        " : nc == 1 ? "ld.global.nc     " : nc == 2 ? "ld.global.nc.v2  " : "ld.global.nc.v4 (256-bit)",
             double(r[0]) / hops);
    }
    cudaFree(d);
    cudaFree(o);
  }
  return 0;
}
