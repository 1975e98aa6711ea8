// DRAM bytes per random 32-byte read vs load flavor (B200).  Offsets are
// precomputed uniform random 32-byte slots of a 4 GiB buffer; one read per
// thread.  Prints time; run under ncu for dram__bytes_read.
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define KERNEL(NAME, ASM)                                                                    \
  __global__ void NAME(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ idx,   \
                       uint64_t count, unsigned long long* sink) {                          \
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;                           \
    if (i >= count) return;                                                                  \
    const uint8_t* p = buf + (uint64_t)idx[i] * 32;                                          \
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;                                                 \
    ASM;                                                                                     \
    if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345) atomicAdd(sink, 1ull);                               \
  }

KERNEL(g_nc256, asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p)))
KERNEL(g_256, asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p)))
KERNEL(g_nc128x2, asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a0), "=l"(a1) : "l"(p)); asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a2), "=l"(a3) : "l"(p + 16)))
KERNEL(g_nc128, asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a0), "=l"(a1) : "l"(p)))
KERNEL(g_nc32, { unsigned v; asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p)); a0 = v; })
KERNEL(g_l2_64, asm volatile("ld.global.nc.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p)))
KERNEL(g_ef, asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(p)))
KERNEL(g_cv, asm volatile("ld.global.cv.v2.u64 {%0,%1}, [%2];" : "=l"(a0), "=l"(a1) : "l"(p)); asm volatile("ld.global.cv.v2.u64 {%0,%1}, [%2];" : "=l"(a2), "=l"(a3) : "l"(p+16)))

typedef void (*kfn)(const uint8_t*, const uint32_t*, uint64_t, unsigned long long*);

int main() {
  const uint64_t total = 4ull << 30, count = 1ull << 25;
  uint8_t* buf; unsigned long long* sink; uint32_t* d_idx;
  cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  cudaMalloc(&sink, 8);
  std::vector<uint32_t> h(count);
  std::mt19937_64 rng(1);
  for (uint64_t i = 0; i < count; ++i) h[i] = uint32_t(rng() % (total / 32));
  cudaMalloc(&d_idx, count * 4);
  cudaMemcpy(d_idx, h.data(), count * 4, cudaMemcpyHostToDevice);
  const char* names[] = {"nc256", "256", "nc128x2", "nc128", "nc32", "l2_64", "evict_first", "cv128x2"};
  kfn fns[] = {g_nc256, g_256, g_nc128x2, g_nc128, g_nc32, g_l2_64, g_ef, g_cv};
  for (int f = 0; f < 8; ++f) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    fns[f]<<<count / 256, 256>>>(buf, d_idx, count, sink);
    cudaEventRecord(e0);
    fns[f]<<<count / 256, 256>>>(buf, d_idx, count, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-12s %.1f us  %.1f G reads/s\n", names[f], ms * 1e3, count / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
