// What does a scattered 32-byte result store cost on B200?  The binned Occ
// step (sort a batch's pairs by index region so each region is served from
// L2) has to write every 32-byte result back at its ORIGINAL position.  Three
// store orders over the same 2^24 sectors (512 MB):
//   dense   : thread i -> sector i
//   random  : thread i -> sector perm(i)
//   phased  : B launches; launch p writes the sectors of class p (a hash of
//             the sector number), in increasing address order — the order a
//             stable partition by index region leaves them in.
// Each thread also reads 12 bytes of a compact (k, l, idx) record, like the
// binned kernel would.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>
#include <cuda_runtime.h>

__global__ void k_store(const uint32_t* __restrict__ idx, uint64_t count, uint4* __restrict__ out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  const uint32_t j = idx[t];
  const uint4 v = make_uint4(j, j + 1, j + 2, j + 3);
  uint4* p = out + 2ull * j;
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + 1), "r"(v.w), "r"(v.z), "r"(v.y), "r"(v.x));
}

static float time_launches(const std::vector<std::pair<const uint32_t*, uint64_t>>& parts, uint4* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    for (auto& p : parts) k_store<<<unsigned((p.second + 255) / 256), 256>>>(p.first, p.second, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best = std::min(best, ms);
  }
  return best;
}

int main() {
  const uint64_t N = 1ull << 24;
  uint4* out;
  cudaMalloc(&out, N * 32);
  std::vector<uint32_t> h(N);
  uint32_t* d;
  cudaMalloc(&d, N * 4);
  auto report = [&](const char* name, float ms) {
    printf("%-28s %8.1f us  %6.1f G sectors/s  %7.1f GB/s stored\n", name, ms * 1e3, N / ms / 1e6, N * 32.0 / ms / 1e6);
  };
  std::iota(h.begin(), h.end(), 0u);
  cudaMemcpy(d, h.data(), N * 4, cudaMemcpyHostToDevice);
  report("dense", time_launches({{d, N}}, out));
  std::mt19937_64 rng(1);
  std::shuffle(h.begin(), h.end(), rng);
  cudaMemcpy(d, h.data(), N * 4, cudaMemcpyHostToDevice);
  report("random", time_launches({{d, N}}, out));
  for (int B : {2, 4, 8, 16, 32, 64}) {
    // class of sector j = a hash of j; phase p holds its sectors in increasing order
    std::vector<std::vector<uint32_t>> cls(B);
    for (uint32_t j = 0; j < N; ++j) cls[(j * 2654435761u >> 7) % B].push_back(j);
    std::vector<std::pair<const uint32_t*, uint64_t>> parts;
    uint64_t off = 0;
    for (int p = 0; p < B; ++p) {
      cudaMemcpy(d + off, cls[p].data(), cls[p].size() * 4, cudaMemcpyHostToDevice);
      parts.push_back({d + off, cls[p].size()});
      off += cls[p].size();
    }
    char name[64];
    snprintf(name, sizeof name, "phased, %d classes", B);
    report(name, time_launches(parts, out));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
