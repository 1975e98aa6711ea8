// B200-native FM-index engine: host side of libfmgpu.so and the C ABI of
// include/fmgpu.h.  Kernels (sm_100a, integer/popcount + random 32-byte
// gathers; no tensor cores — the Occ step has no GEMM shape):
//   kernels_occ.cuh      k_build_lines, k_occ_pair (+ 2-lane, wide-line coop),
//                        k_random_fetch                        (occ.py:59-96)
//   kernels_search.cuh   k_exact, k_psi, k_locate              (search.py:74-94, 172-208)
//   kernels_inexact.cuh  k_dbound, k_inexact (DFS), k_spine / k_chain (z = 1),
//                        sort / dedup / gather                 (search.py:97-159)
//   kernels_bidir.cuh    bidirectional z = 1 engines (split DFS, level-synchronous)
//   kernels_flat.cuh     flat z = 1 engine: k_flat_probe / _extend / _collect over the one-edit neighbourhood, presence filter

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <string>
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <array>
#include <chrono>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "fmgpu_internal.h"
#include "occ_device.cuh"

namespace fmg {

thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

#define FMG_CK(expr)                                                                      \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::fmg::CudaError(std::string(#expr) + " failed: " + cudaGetErrorString(e_)); \
  } while (0)

#define FMG_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) throw std::invalid_argument(msg); \
  } while (0)

// Restores the caller's current device on scope exit (the library must not
// disturb torch's or the application's device selection).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    FMG_CK(cudaGetDevice(&prev));
    if (prev != dev) FMG_CK(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Allocation size handed to the stream-ordered pool: sizes of 64 MiB and
// up are rounded up to a multiple of 64 MiB, so per-call buffers whose
// exact size drifts from call to call (result sets) map to the same pool
// blocks instead of growing the pool — measured on B200: an 800 MB result
// buffer a few MB larger than any free block cost 100-300 ms of mapping.
inline size_t pool_bytes(size_t bytes) {
  const size_t g = size_t(64) << 20;
  return bytes >= g ? (bytes + g - 1) / g * g : bytes;
}

// ---------------------------------------------------------------------------
// Guard mode (FMG_GUARD=1): every library allocation gets its own virtual
// address range with unmapped guard space on both sides, and ends exactly at
// its mapped end, so an out-of-bounds access by any kernel faults (illegal
// address) instead of reading a neighbour.  The bounds-checking substitute
// for compute-sanitizer, which this pool does not allow (tools/guard_check.sh).
// Allocation and free become synchronous; production runs never set it.
// ---------------------------------------------------------------------------
bool guard_mode() {
  static const bool on = [] {
    const char* e = std::getenv("FMG_GUARD");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

struct GuardRec {
  CUdeviceptr va;
  size_t reserved, mapped;
  CUmemGenericAllocationHandle h;
};
std::mutex g_guard_mu;
std::unordered_map<void*, GuardRec> g_guard;

// The driver's virtual-memory API, resolved from libcuda at run time (the
// library must load on hosts without a driver, e.g. the CPU build check).
struct CuVmm {
  CUresult (*gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*release)(CUmemGenericAllocationHandle);
  CUresult (*addr_free)(CUdeviceptr, size_t);
};
const CuVmm& cu_vmm() {
  static const CuVmm v = [] {
    CuVmm r{};
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error("FMG_GUARD=1 needs libcuda.so.1");
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f) throw std::runtime_error(std::string("libcuda lacks ") + n);
      return f;
    };
    r.gran = reinterpret_cast<decltype(r.gran)>(sym("cuMemGetAllocationGranularity"));
    r.reserve = reinterpret_cast<decltype(r.reserve)>(sym("cuMemAddressReserve"));
    r.create = reinterpret_cast<decltype(r.create)>(sym("cuMemCreate"));
    r.map = reinterpret_cast<decltype(r.map)>(sym("cuMemMap"));
    r.access = reinterpret_cast<decltype(r.access)>(sym("cuMemSetAccess"));
    r.unmap = reinterpret_cast<decltype(r.unmap)>(sym("cuMemUnmap"));
    r.release = reinterpret_cast<decltype(r.release)>(sym("cuMemRelease"));
    r.addr_free = reinterpret_cast<decltype(r.addr_free)>(sym("cuMemAddressFree"));
    return r;
  }();
  return v;
}

#define FMG_CU(expr)                                                                  \
  do {                                                                                \
    CUresult r_ = (expr);                                                             \
    if (r_ != CUDA_SUCCESS) throw ::fmg::CudaError(std::string(#expr) + " failed"); \
  } while (0)

void* guarded_alloc(size_t bytes) {
  int dev = 0;
  FMG_CK(cudaGetDevice(&dev));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gran = 0;
  const CuVmm& cu = cu_vmm();
  FMG_CU(cu.gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  // 32-byte granularity keeps the 256-bit vector loads aligned; an access
  // past the 32-byte-rounded end of the buffer faults
  const size_t want = std::max<size_t>((bytes + 31) / 32 * 32, 32);
  const size_t mapped = (want + gran - 1) / gran * gran;
  GuardRec r{};
  r.reserved = mapped + 2 * gran;
  r.mapped = mapped;
  FMG_CU(cu.reserve(&r.va, r.reserved, gran, 0, 0));
  FMG_CU(cu.create(&r.h, mapped, &prop, 0));
  FMG_CU(cu.map(r.va + gran, mapped, 0, r.h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  FMG_CU(cu.access(r.va + gran, mapped, &acc, 1));
  void* p = reinterpret_cast<void*>(r.va + gran + (mapped - want));  // ends at the guard page
  std::lock_guard<std::mutex> lock(g_guard_mu);
  g_guard[p] = r;
  return p;
}

void guarded_free(void* p) {
  GuardRec r;
  {
    std::lock_guard<std::mutex> lock(g_guard_mu);
    auto it = g_guard.find(p);
    if (it == g_guard.end()) return;
    r = it->second;
    g_guard.erase(it);
  }
  const CuVmm& cu = cu_vmm();
  cu.unmap(r.va + (r.reserved - r.mapped) / 2, r.mapped);
  cu.release(r.h);
  cu.addr_free(r.va, r.reserved);
}

// Bumped by every synchronous allocation / free of this library: available_bytes()
// re-reads the device's free memory only after one of them (or after 250 ms).
std::atomic<uint64_t> g_mem_epoch{1};

// Synchronous allocations of the index structures (lines, chunks, tables).
cudaError_t dmalloc_v(void** p, size_t bytes) {
  g_mem_epoch.fetch_add(1, std::memory_order_relaxed);
  if (!guard_mode()) return cudaMalloc(p, bytes);
  try {
    *p = guarded_alloc(bytes);
    return cudaSuccess;
  } catch (...) {
    return cudaErrorMemoryAllocation;
  }
}
template <typename T>
cudaError_t dmalloc(T** p, size_t bytes) {
  return dmalloc_v(reinterpret_cast<void**>(p), bytes);
}
void dfree(void* p) {
  if (!p) return;
  g_mem_epoch.fetch_add(1, std::memory_order_relaxed);
  if (!guard_mode()) {
    cudaFree(p);
    return;
  }
  cudaDeviceSynchronize();
  guarded_free(p);
}

// Stream-ordered scratch / result allocations (pool-backed, cheap after warm-up).
cudaError_t amalloc(void** p, size_t bytes, cudaStream_t s) {
  if (!guard_mode()) return cudaMallocAsync(p, pool_bytes(bytes), s);
  cudaStreamSynchronize(s);
  return dmalloc_v(p, bytes);
}
void afree(void* p, cudaStream_t s) {
  if (!p) return;
  if (!guard_mode()) {
    cudaFreeAsync(p, s);
    return;
  }
  cudaDeviceSynchronize();
  guarded_free(p);
}

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t s) : stream(s) {
    if (count) FMG_CK(amalloc(reinterpret_cast<void**>(&ptr), count * sizeof(T), s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), stream(o.stream) { o.ptr = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(ptr, o.ptr);
    std::swap(stream, o.stream);
    return *this;
  }
  ~DevBuf() {
    if (ptr) afree(ptr, stream);
  }
};

}  // namespace fmg

#include "kernels_occ.cuh"
#include "kernels_search.cuh"
#include "kernels_inexact.cuh"
#include "kernels_bidir.cuh"
#include "kernels_flat.cuh"
#include "kernels_bucket.cuh"
#include "kernels_chunk.cuh"

namespace fmg {

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------

int sm_count(int device) {
  int v = 0;
  FMG_CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

size_t available_bytes_now(int device);

// Memory a call may size its scratch from: device free memory plus what the
// stream-ordered pool holds but is not using.  Unlike cudaMemGetInfo alone
// this does not shrink as the pool keeps freed blocks (release threshold is
// unlimited), so scratch sizes stay the same from call to call and the pool
// reuses its blocks instead of mapping fresh memory (measured on B200: the
// config-2 z = 1 call varied 8 -> 50 ms while sizes followed cudaMemGetInfo).
size_t available_bytes(int device) {
  // cudaMemGetInfo is a slow driver call (and run_inexact asks three times per
  // search): the answer is kept for 250 ms unless this library allocated or
  // freed device memory synchronously in between
  struct Cached {
    size_t value = 0;
    uint64_t epoch = 0;
    std::chrono::steady_clock::time_point at{};
  };
  static std::mutex cache_mu;
  static std::unordered_map<int, Cached> cached;
  const uint64_t epoch = g_mem_epoch.load(std::memory_order_relaxed);
  const auto now = std::chrono::steady_clock::now();
  {
    std::lock_guard<std::mutex> lock(cache_mu);
    const Cached& c = cached[device];
    static const int keep_ms = [] {  // FMG_AVAIL_CACHE_MS (A/B; 0: ask the driver every time)
      const char* e = std::getenv("FMG_AVAIL_CACHE_MS");
      return e ? std::atoi(e) : 250;
    }();
    if (c.value && c.epoch == epoch && now - c.at < std::chrono::milliseconds(keep_ms)) return c.value;
  }
  const size_t fresh = available_bytes_now(device);
  std::lock_guard<std::mutex> lock(cache_mu);
  cached[device] = Cached{fresh, epoch, now};
  return fresh;
}

size_t available_bytes_now(int device) {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return size_t(8) << 30;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
      free_b += size_t(reserved - used);
  }
  // round down to 1 GiB, and keep the previous figure unless memory got
  // >10% tighter or >50% roomier: another process freeing its memory while
  // this one runs (the previous test or bench on the box) must not change
  // the sizes on every call — each change remaps GBs of pool memory
  // (measured: config 2 at 3.6 vs 16 ms per call for a whole process)
  const size_t g = size_t(1) << 30;
  const size_t cur = free_b > g ? free_b / g * g : free_b;
  static std::mutex mu;
  static std::unordered_map<int, size_t> last;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = last[device];
  if (c == 0 || cur < c / 10 * 9 || cur > c / 2 * 3) c = cur;
  return c;
}

}  // namespace fmg

struct fmg_index {
  int device = 0;
  uint64_t n = 0, sentinel_row = 0, c[5] = {0, 0, 0, 0, 0};
  uint64_t n_buckets = 0, n_lines = 0, n_samples = 0;
  int words = 2;  // line layout: W words of 32 chars per line (occ_device.cuh)
  uint8_t* lines = nullptr;
  // 128-byte chunk layout of the same transform (kernels_chunk.cuh), built
  // for HBM-resident indexes only: the Occ-step kernel reads it instead of
  // the lines (416 instead of 256 characters per DRAM fetch)
  uint32_t* chunks = nullptr;
  uint64_t n_chunks = 0;
  int chunk_sectors = 4;  // 4: 128-byte chunks; 2: 64-byte chunks read with the L2::64B hint
  // Attachments (fmg_index_set_samples / fmg_index_set_reverse) are
  // one-time: the first attach uploads and publishes the pointer with a
  // release store under attach_mu, later attaches are no-ops, and nothing is
  // freed before fmg_index_destroy — a launch that read a pointer can never
  // see it freed or replaced.  Readers use acquire loads.
  std::mutex attach_mu;
  std::atomic<uint32_t*> samples{nullptr};
  int sms = 148;
  // exact-search k-mer table (built on first large exact call; see KmerTable)
  std::mutex lut_mu;
  uint2* lut = nullptr;
  uint32_t lut_k = 0;
  // optional index of the reversed text (fmg_index_set_reverse): the
  // bidirectional z = 1 engine (kernels_bidir.cuh) and its prefix table
  std::atomic<uint8_t*> rev_lines{nullptr};
  uint64_t rev_sentinel_row = 0;
  uint2* lut_r = nullptr;
  uint32_t tail[16] = {};
  // exact-search k-mer table one level beyond the prefix table (level
  // lut_k + 1 alone; see kmer_table), or null
  uint2* lut_x = nullptr;
  uint32_t lut_x_k = 0;
  bool lut_x_tried = false;
  // presence filter of the flat z = 1 engine (kernels_flat.cuh FlatFilter):
  // NO bitmaps of 4^B bits, built on first use from the level-lut_x_k table
  uint32_t* flt_bits = nullptr;
  uint32_t flt_B = 0, flt_G = 0, flt_NO = 0;
  bool flt_tried = false;
  // dedup hash table of the inexact engines, kept between calls with a
  // monotone epoch so it is zeroed only when allocated or when the epochs
  // wrap (EpochTable)
  std::mutex ep_mu;
  uint4* ep_table = nullptr;
  uint64_t ep_entries = 0;
  uint64_t ep_next = 1;

  fmg::IndexView view_rev() const {
    fmg::IndexView v = view();
    v.lines = rev_lines.load(std::memory_order_acquire);
    v.samples = nullptr;
    v.sentinel_row = uint32_t(rev_sentinel_row);
    return v;
  }

  fmg::IndexView view() const {
    fmg::IndexView v;
    v.lines = lines;
    v.samples = samples.load(std::memory_order_acquire);
    v.n = uint32_t(n);
    v.sentinel_row = uint32_t(sentinel_row);
    for (int s = 0; s < 5; ++s) v.c[s] = uint32_t(c[s]);
    return v;
  }
};

struct fmg_matches {
  int device = 0;
  uint64_t patterns = 0, total = 0, steps = 0, lines = 0;  // work counters: Occ steps, lines fetched
  uint64_t launches = 0;  // kernels of this library the search launched (flat engine; 0 = not counted)
  uint64_t* row_off = nullptr;  // device, patterns + 1
  uint32_t* k = nullptr;        // device, total
  uint32_t* l = nullptr;
  uint64_t* kl = nullptr;       // or: device, k << 32 | l packed (host-sync-free engine); split on copy
  uint8_t* diffs = nullptr;
  cudaStream_t stream = nullptr;  // the stream the search ran on (buffers are freed on it)
};

namespace {

using namespace fmg;

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Line layout.  W = 2 (32-byte lines, one sector per Occ) is the default for
// every index size: measured on B200, a random L2 miss costs one DRAM request
// (~48 G requests/s chip-wide) whatever its size up to 64 B, and W = 6 / 14
// lines read by one thread need 2-4 requests and 3-7x the popcount work
// (tools/size_sweep.py, profiles/).  FMG_LINE_WORDS=2|6|14 overrides (the
// tests exercise every layout).
int choose_words(uint64_t n_buckets) {
  if (const char* env = std::getenv("FMG_LINE_WORDS")) {
    const int w = std::atoi(env);
    FMG_REQUIRE(w == 2 || w == 6 || w == 14, "FMG_LINE_WORDS must be 2, 6 or 14");
    return w;
  }
  (void)n_buckets;
  return 2;
}

void check_index(const fmg_index* ix) { FMG_REQUIRE(ix != nullptr, "null index handle"); }

// Input-error word of ONE host-buffer call (status bits: 1 = position out of
// range or pair out of order, 2 = predecessor walk did not terminate), from
// the stream-ordered pool, so no call ever sees another call's errors.
// Device entry points instead pass the caller's own status word straight to
// the kernels (NULL: unchecked, the kernels skip the report).
struct CallStatus {
  DevBuf<uint32_t> own;
  uint32_t* word = nullptr;
  CallStatus(uint32_t* caller, cudaStream_t s) {
    if (caller) {
      word = caller;
    } else {
      own = DevBuf<uint32_t>(1, s);
      word = own.ptr;
      FMG_CK(cudaMemsetAsync(word, 0, sizeof(uint32_t), s));
    }
  }
  // Reads this call's word after everything queued on `s` (synchronises).
  void raise_if_set(cudaStream_t s, const char* what) {
    uint32_t h = 0;
    FMG_CK(cudaMemcpyAsync(&h, word, sizeof(h), cudaMemcpyDeviceToHost, s));
    FMG_CK(cudaStreamSynchronize(s));
    if (h & 2u) throw std::runtime_error("predecessor walk did not terminate; index is corrupt");
    if (h) throw std::invalid_argument(what);
  }
};

// Runs f(std::integral_constant<int, W>) for the index's line layout.
template <typename F>
void with_words(const fmg_index* ix, F&& f) {
  switch (ix->words) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 14: f(std::integral_constant<int, 14>{}); break;
    default: throw std::invalid_argument("unsupported line layout");
  }
}

constexpr int kOccPer = 1;

// FMG_OCC_CHUNK=0: Occ steps read the lines even when chunks exist (A/B hook)
bool chunk_off() {
  static const bool off = [] {
    const char* e = std::getenv("FMG_OCC_CHUNK");
    return e != nullptr && std::atoi(e) == 0;
  }();
  return off;
}

// Chunk layout for line arrays above this size (HBM-resident; the L2-resident
// config 1 keeps the one-sector lines, whose bound is the L2 request rate).
// FMG_CHUNK_MIN_BYTES overrides (tests build chunks for small indexes too).
uint64_t chunk_min_line_bytes() {
  const char* e = std::getenv("FMG_CHUNK_MIN_BYTES");
  return e ? std::strtoull(e, nullptr, 10) : (uint64_t(64) << 20);
}

// ... and up to this size: beyond ~2 Gbp the chunk kernel's four sector
// requests per step lose to the lines' one or two (3.1 Gbp synthetic, 2^24
// config-1 pairs: chunks 723-774 us, lines 535 us; profiles/r02_occ_layout.md).
// FMG_CHUNK_MAX_BYTES overrides.
uint64_t chunk_max_line_bytes() {
  const char* e = std::getenv("FMG_CHUNK_MAX_BYTES");
  return e ? std::strtoull(e, nullptr, 10) : (uint64_t(1) << 30);
}

// Sectors per chunk of the Occ-step layout: FMG_CHUNK_SECTORS=2|4 (A/B).
int chunk_sectors_default() {
  const char* e = std::getenv("FMG_CHUNK_SECTORS");
  const int v = e ? std::atoi(e) : 4;
  FMG_REQUIRE(v == 2 || v == 4, "FMG_CHUNK_SECTORS must be 2 or 4");
  return v;
}

uint32_t* build_chunks(const fmg_index* ix, const void* bucket_records, uint64_t& n_chunks) {
  const int ns = ix->chunk_sectors;
  const uint64_t chars = ns == 2 ? fmg::ChunkTraits<2>::kChars : fmg::ChunkTraits<4>::kChars;
  n_chunks = (ix->n + 1 + chars - 1) / chars;
  uint32_t* chunks = nullptr;
  FMG_CK(dmalloc(&chunks, n_chunks * 32 * ns));
  uint64_t* staging = nullptr;
  const uint64_t nb = ix->n_buckets;
  cudaError_t e = cudaMalloc(&staging, nb * 64 + 64);
  uint32_t bad = 0;
  if (e == cudaSuccess) {
    uint32_t* err = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(staging) + nb * 64);
    e = cudaMemcpy(staging, bucket_records, nb * 64, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(err, 0, 4);
    if (e == cudaSuccess) {
      if (ns == 2)
        fmg::k_build_chunks<2><<<unsigned((n_chunks + 255) / 256), 256>>>(staging, nb, chunks, n_chunks, err);
      else
        fmg::k_build_chunks<4><<<unsigned((n_chunks + 255) / 256), 256>>>(staging, nb, chunks, n_chunks, err);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&bad, err, 4, cudaMemcpyDeviceToHost);
    cudaFree(staging);
  }
  if (e != cudaSuccess || bad) dfree(chunks);
  FMG_CK(e);
  FMG_REQUIRE(bad == 0, "bucket base does not fit 32 bits");
  return chunks;
}

template <int PER>
void launch_occ_pair_t(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, cudaStream_t s,
                       uint32_t* err, int threads) {
  const uint64_t per_block = uint64_t(threads) * PER;
  const uint64_t blocks = (count + per_block - 1) / per_block;
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    // two lanes per step only for HBM-resident line arrays (> 64 MB): +4% on
    // config 1-H, -8% on the L2-resident config 1 (profiles/r01_occ.md)
    const char* e2l = std::getenv("FMG_OCC_2LANE");  // A/B hook
    const bool two_lane = e2l ? std::atoi(e2l) != 0 : ix->n_lines * 32ull > (64ull << 20);
    if (ix->chunks && !chunk_off()) {
      if (ix->chunk_sectors == 2)
        k_occ_pair_chunk<2><<<dim3(unsigned((count + 255) / 256)), 256, 0, s>>>(
            ix->view(), ix->chunks, reinterpret_cast<const uint2*>(kl), count, out, err);
      else
        k_occ_pair_chunk<4><<<dim3(unsigned((count + 255) / 256)), 256, 0, s>>>(
            ix->view(), ix->chunks, reinterpret_cast<const uint2*>(kl), count, out, err);
    } else if (W == 2 && two_lane) {
      static const bool bulk2 = [] {  // FMG_OCC_BULK=1: bulk-copy stores (A/B; slower with two lanes per step on config 1)
        const char* e = std::getenv("FMG_OCC_BULK");
        return e != nullptr && std::atoi(e) != 0;
      }();
      if (bulk2 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0)
        k_occ_pair_2l<true><<<dim3(unsigned((2 * count + 255) / 256)), 256, 0, s>>>(
            ix->view(), reinterpret_cast<const uint2*>(kl), count, out, err);
      else
        k_occ_pair_2l<false><<<dim3(unsigned((2 * count + 255) / 256)), 256, 0, s>>>(
            ix->view(), reinterpret_cast<const uint2*>(kl), count, out, err);
    } else if (W == 2) {
      // counts leave through one bulk copy per block: 90.6 vs 89.2 G steps/s on
      // config 1 (profiles/r02_ab_occ_bulk.log); FMG_OCC_BULK=0: per-thread stores (A/B)
      static const bool bulk = [] {
        const char* e = std::getenv("FMG_OCC_BULK");
        return e == nullptr || std::atoi(e) != 0;
      }();
      static const bool exch = [] {  // FMG_OCC_EXCH=1: neighbouring lanes fetch each other's lines (A/B: 85.9 vs 90.5 G steps/s, off)
        const char* e = std::getenv("FMG_OCC_EXCH");
        return e != nullptr && std::atoi(e) != 0;
      }();
      if (PER == 1 && bulk && exch && (reinterpret_cast<uintptr_t>(out) & 15u) == 0)
        k_occ_pair<1, 2, true, true><<<dim3(unsigned(blocks)), threads, 0, s>>>(
            ix->view(), reinterpret_cast<const uint2*>(kl), count, out, err);
      else if (PER == 1 && bulk && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
        // FMG_OCC_DYNSMEM=bytes: unused dynamic shared memory, to cap the resident blocks per SM (A/B)
        static const size_t pad = [] {
          const char* e = std::getenv("FMG_OCC_DYNSMEM");
          return e ? size_t(std::atoi(e)) : size_t(0);
        }();
        k_occ_pair<1, W, true><<<dim3(unsigned(blocks)), threads, pad, s>>>(
            ix->view(), reinterpret_cast<const uint2*>(kl), count, out, err);
      }
      else
        k_occ_pair<PER, W><<<dim3(unsigned(blocks)), threads, 0, s>>>(ix->view(), reinterpret_cast<const uint2*>(kl),
                                                                        count, out, err);
    } else {  // wide lines: lane-cooperative, persistent grid-stride
      constexpr int LANES = int(LineTraits<W>::kBytes / 32);
      const uint64_t nb = (count * LANES + 255) / 256;
      k_occ_pair_coop<W><<<dim3(unsigned(std::max<uint64_t>(nb, 1))), 256, 0, s>>>(
          ix->view(), reinterpret_cast<const uint2*>(kl), count, out, err);
    }
  });
  FMG_CK(cudaGetLastError());
}

void launch_occ_pair(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, cudaStream_t s,
                     uint32_t* err, int per = kOccPer, int threads = 128) {
  if (count == 0) return;
  FMG_REQUIRE(threads == 64 || threads == 128 || threads == 256, "threads must be 64, 128 or 256");
  switch (per) {
    case 1: launch_occ_pair_t<1>(ix, kl, count, out, s, err, threads); break;
    case 2: launch_occ_pair_t<2>(ix, kl, count, out, s, err, threads); break;
    case 4: launch_occ_pair_t<4>(ix, kl, count, out, s, err, threads); break;
    default: throw std::invalid_argument("per must be 1, 2 or 4");
  }
}

// Resident blocks per SM of (kernel, threads, dynamic smem), cached: the
// occupancy query costs about a microsecond of host time, which small
// latency-bound batches (config 0: 23 us per call) cannot hide.
int blocks_per_sm(const void* kernel, int threads, size_t smem) {
  struct Key {
    const void* k;
    int t;
    size_t s;
    bool operator==(const Key& o) const { return k == o.k && t == o.t && s == o.s; }
  };
  struct Hash {
    size_t operator()(const Key& x) const {
      return std::hash<const void*>()(x.k) ^ (size_t(x.t) << 40) ^ (x.s << 8);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, int, Hash> cache;
  int dev = 0;
  FMG_CK(cudaGetDevice(&dev));
  const Key key{kernel, threads * 64 + dev, smem};  // one entry per device (same GPU model in practice)
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = per_sm;
  return per_sm;
}

unsigned persistent_blocks(const fmg_index* ix, const void* kernel, int threads, uint64_t work) {
  const int per_sm = blocks_per_sm(kernel, threads, 0);
  static const int mult = [] {
    const char* e = std::getenv("FMG_GRID_MULT");  // tuning hook: waves of the persistent grid
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  uint64_t blocks = uint64_t(std::max(per_sm, 1)) * ix->sms * mult;
  const uint64_t need = (work + threads - 1) / threads;
  return unsigned(std::max<uint64_t>(1, std::min(blocks, need)));
}

// Grid for the lane-refill search kernels: about kPerThread queries per
// thread, i.e. many more blocks than fit at once.  Measured on B200 (config
// 4, tools/prof_exact.py): letting the block scheduler refill SMs beats a
// persistent one-wave grid whose lanes refill themselves (2.56 -> 3.3 G
// seeds/s), because a self-refilling lane stalls the rest of its warp.
unsigned wave_blocks(const fmg_index* ix, const void* kernel, int threads, uint64_t work) {
  constexpr uint64_t kPerThread = 4;
  const uint64_t resident = persistent_blocks(ix, kernel, threads, work);
  const uint64_t waves = (work + threads * kPerThread - 1) / (threads * kPerThread);
  return unsigned(std::min<uint64_t>(std::max<uint64_t>(resident, waves), 1u << 30));
}

// The prefix interval table of the index (PrefixTable), built on first use
// by a large call (>= 1024 patterns): levels 1..K, level j built from level
// j-1 with one Occ step per entry (k_lut_level), 8 * (4^(K+1) - 4) / 3 bytes.
// K = clamp(floor(log4 n) + 1, 4, 15), lowered while the table would take
// more than a quarter of the free device memory: 11.5 GB at K = 15 (1 and
// 3.1 Gbp), 716 MB at K = 13 (64 Mbp).  Measured on config 4 (2^28 20-mers,
// 1 Gbp): K = 12 / 13 / 14 / 15 -> 6.45 / 7.40 / 8.54 / 10.04 G seeds/s,
// table build 13 ms at K = 15 — HBM capacity spent to skip dependent steps.  Level K is the
// exact-search k-mer table (KmerTable): its entries are what exact_search
// returns for each K-mer, first empty interval included.  FMG_EXACT_LUT=0
// disables both uses, FMG_LUT_K=j forces K (A/B).
constexpr int kLutBias = 1;
constexpr uint32_t kLutMax = 15;

void build_prefix_levels(const fmg_index* ix, const fmg::IndexView& v, uint2* lut, int k, cudaStream_t s) {
  for (int j = 1; j <= k; ++j) {
    const uint64_t cnt = uint64_t(1) << (2 * j);
    const uint2* parent = j == 1 ? nullptr : lut + PrefixTable::off64(j - 1);
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      k_lut_level<W><<<unsigned((cnt + 255) / 256), 256, 0, s>>>(v, parent, lut + PrefixTable::off64(j), cnt);
    });
    FMG_CK(cudaGetLastError());
  }
}

PrefixTable prefix_table(const fmg_index* cix, uint64_t count, cudaStream_t s) {
  static const bool enabled = [] {
    const char* e = std::getenv("FMG_EXACT_LUT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (!enabled || count < 1024) return {};
  auto* ix = const_cast<fmg_index*>(cix);  // the table is a cache; the index itself never changes
  std::lock_guard<std::mutex> lock(ix->lut_mu);
  if (!ix->lut) {
    int k = 0;
    while ((uint64_t(1) << (2 * (k + 1))) <= ix->n) ++k;  // floor(log4 n)
    k = std::min<int>(int(kLutMax), std::max<int>(4, k + kLutBias));
    if (const char* e = std::getenv("FMG_LUT_K")) k = std::min<int>(15, std::max<int>(1, std::atoi(e)));  // A/B
    size_t free_b = 0, total_b = 0;
    FMG_CK(cudaMemGetInfo(&free_b, &total_b));
    while (k > 1 && PrefixTable::off64(k + 1) * sizeof(uint2) > free_b / 4) --k;
    uint2* lut = nullptr;
    FMG_CK(dmalloc(&lut, PrefixTable::off64(k + 1) * sizeof(uint2)));
    build_prefix_levels(ix, ix->view(), lut, k, s);
    FMG_CK(cudaStreamSynchronize(s));
    ix->lut = lut;
    ix->lut_k = uint32_t(k);
  }
  return PrefixTable{ix->lut, ix->lut_k};
}

// The reverse index's prefix table, same K as the forward one (empty when
// there is no reverse index, no forward table, or no room for it).
PrefixTable prefix_table_rev(const fmg_index* cix, uint64_t count, cudaStream_t s) {
  const PrefixTable tf = prefix_table(cix, count, s);
  if (!tf.base || !cix->rev_lines.load(std::memory_order_acquire)) return {};
  auto* ix = const_cast<fmg_index*>(cix);
  std::lock_guard<std::mutex> lock(ix->lut_mu);
  if (!ix->lut_r) {
    const uint64_t bytes = PrefixTable::off64(tf.k + 1) * sizeof(uint2);
    size_t free_b = 0, total_b = 0;
    FMG_CK(cudaMemGetInfo(&free_b, &total_b));
    if (bytes > free_b / 3) return {};
    uint2* lut = nullptr;
    FMG_CK(dmalloc(&lut, bytes));
    build_prefix_levels(ix, ix->view_rev(), lut, int(tf.k), s);
    FMG_CK(cudaStreamSynchronize(s));
    ix->lut_r = lut;
  }
  return PrefixTable{ix->lut_r, tf.k};
}

// The exact search's k-mer table.  Exact search needs only the last level,
// so it goes beyond the prefix table (to level floor(log4 n) + 4, at most
// 16 so keys stay 32-bit) when the level fits in a quarter of the available
// memory: level 16 is 34.4 GB, built from level 15 with one Occ step per
// entry.  Patterns shorter than that level use the prefix table's level of
// their own length (the exact answer in one gather) or its level K.  Measured on config 4 (2^28 x 20 bp, 1 Gbp): K = 15 -> 16
// takes present seeds from 5 to 4 dependent steps and most random seeds to
// an empty interval in the table.  FMG_EXACT_LUT_EXT=0 disables it (A/B).
// Level of the exact search's own k-mer table: floor(log4 n) + 4, at most 16
// and at least K + 1.  Small indexes go further past the prefix table, whose
// K tracks log4 n for the inexact engines' sake — config 0 (1 Mbp): K = 10,
// exact level 13 (537 MB), two dependent steps fewer per 32-bp pattern;
// genome-scale indexes stop at 16.
uint32_t exact_table_level(const fmg_index* ix, const PrefixTable& pt) {
  int lg = 0;
  while ((uint64_t(1) << (2 * (lg + 1))) <= ix->n) ++lg;  // floor(log4 n)
  return std::min<uint32_t>(16, std::max<uint32_t>(pt.k + 1, uint32_t(lg + 4)));
}

KmerTable kmer_table(const fmg_index* cix, uint64_t count, cudaStream_t s) {
  const PrefixTable pt = prefix_table(cix, count, s);
  if (!pt.base) return {};
  static const bool ext_enabled = [] {
    const char* e = std::getenv("FMG_EXACT_LUT_EXT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  auto* ix = const_cast<fmg_index*>(cix);  // a cache, like the prefix table
  if (ext_enabled) {
    std::lock_guard<std::mutex> lock(ix->lut_mu);
    if (!ix->lut_x_tried) {
      ix->lut_x_tried = true;
      const uint32_t kx = exact_table_level(ix, pt);
      const uint64_t cnt = uint64_t(1) << (2 * kx);
      if (kx <= 16 && cnt * sizeof(uint2) <= available_bytes(ix->device) / 4) {
        uint2* lx = nullptr;
        if (dmalloc(&lx, cnt * sizeof(uint2)) == cudaSuccess) {
          // levels K + 1 .. kx, each from the previous; only the last is kept
          DevBuf<uint2> tmp[2];
          const uint2* parent = pt.base + PrefixTable::off64(pt.k);
          for (uint32_t j = pt.k + 1; j <= kx; ++j) {
            const uint64_t cj = uint64_t(1) << (2 * j);
            uint2* dst = lx;
            if (j < kx) {
              tmp[j & 1] = DevBuf<uint2>(cj, s);
              dst = tmp[j & 1].ptr;
            }
            with_words(ix, [&](auto wt) {
              constexpr int W = decltype(wt)::value;
              k_lut_level<W><<<unsigned((cj + 255) / 256), 256, 0, s>>>(ix->view(), parent, dst, cj);
            });
            FMG_CK(cudaGetLastError());
            parent = dst;
          }
          FMG_CK(cudaStreamSynchronize(s));
          ix->lut_x = lx;
          ix->lut_x_k = kx;
        } else {
          cudaGetLastError();  // clear the failed allocation; keep level K
        }
      }
    }
    if (ix->lut_x) return KmerTable{ix->lut_x, ix->lut_x_k, pt.base, pt.k};
  }
  return KmerTable{pt.base + PrefixTable::off64(pt.k), pt.k, pt.base, pt.k};
}

// Block size of the exact kernels: small batches (config 0: 10,000
// patterns) in 64-thread blocks so every SM gets some of the dependent
// chains instead of 40 blocks of 256 on 40 SMs.
int exact_block_threads(const fmg_index* ix, uint64_t count) {
  return count < uint64_t(ix->sms) * 1024u ? 64 : 256;
}

void launch_exact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, uint32_t* kl_out,
                         cudaStream_t s, unsigned long long* steps) {
  if (count == 0) return;
  PackedPatterns pp{packed, m};
  CodePatterns cp{nullptr, nullptr};
  const KmerTable kt = kmer_table(ix, count, s);
  const int nt = exact_block_threads(ix, count);
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)k_exact<true, W>, nt, count);
    k_exact<true, W><<<blocks, nt, 0, s>>>(ix->view(), pp, cp, count, reinterpret_cast<uint2*>(kl_out), steps, kt);
  });
  FMG_CK(cudaGetLastError());
}

void launch_exact_codes(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                        uint32_t* kl_out, cudaStream_t s, unsigned long long* steps) {
  if (count == 0) return;
  PackedPatterns pp{nullptr, 0};
  CodePatterns cp{codes, offsets};
  const KmerTable kt = kmer_table(ix, count, s);
  const int nt = exact_block_threads(ix, count);
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)k_exact<false, W>, nt, count);
    k_exact<false, W><<<blocks, nt, 0, s>>>(ix->view(), pp, cp, count, reinterpret_cast<uint2*>(kl_out), steps,
                                            kt);
  });
  FMG_CK(cudaGetLastError());
}

void launch_locate(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos, cudaStream_t s,
                   uint32_t* err) {
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    const unsigned blocks = wave_blocks(ix, (const void*)fmg::k_locate<W>, 256, count);
    fmg::k_locate<W><<<blocks, 256, 0, s>>>(ix->view(), rows, count, out_pos, err);
  });
  FMG_CK(cudaGetLastError());
}

// Validates a device pattern batch (k_check_patterns) and returns the
// longest pattern; throws invalid_argument like the reference's ValueErrors.
uint64_t validate_patterns_device(const uint8_t* codes, const uint64_t* offsets, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  DevBuf<unsigned long long> ml(1, s);
  DevBuf<uint32_t> err(1, s);
  FMG_CK(cudaMemsetAsync(ml.ptr, 0, 8, s));
  FMG_CK(cudaMemsetAsync(err.ptr, 0, 4, s));
  k_check_patterns<<<unsigned((count + 255) / 256), 256, 0, s>>>(codes, offsets, count, ml.ptr, err.ptr);
  FMG_CK(cudaGetLastError());
  unsigned long long h_ml = 0;
  uint32_t h_err = 0;
  FMG_CK(cudaMemcpyAsync(&h_ml, ml.ptr, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaMemcpyAsync(&h_err, err.ptr, 4, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  FMG_REQUIRE(!(h_err & 4u), "pattern offsets must start at 0");
  FMG_REQUIRE(!(h_err & 1u), "pattern is empty");
  FMG_REQUIRE(!(h_err & 2u), "symbol code outside [0, 4)");
  return h_ml;
}


// The inexact engines' dedup table for one launch: `entries` uint4 slots
// whose current contents all carry epochs <= epoch0, and room for
// `epochs` more per thread.  The index's persistent table is leased when
// free (zeroed only when (re)allocated or when the epochs would wrap; a
// 1.1 GB memset per launch was 10% of a config-2 call); a concurrent call
// gets a zeroed table of its own.
struct EpochTable {
  uint4* ptr = nullptr;
  uint32_t epoch0 = 0;
  DevBuf<uint4> own;
  std::unique_lock<std::mutex> lease;
};

void lease_epoch_table(fmg_index* ix, uint64_t entries, uint64_t epochs, cudaStream_t s, EpochTable& t) {
  std::unique_lock<std::mutex> lk(ix->ep_mu, std::try_to_lock);
  // only first-pass sized tables (<= 2 GiB) are kept; retry passes with
  // grown capacities get their own
  if (!lk.owns_lock() || epochs >= 0x7FFFFFFFull || entries * sizeof(uint4) > (size_t(2) << 30)) {
    t.own = DevBuf<uint4>(entries, s);
    FMG_CK(cudaMemsetAsync(t.own.ptr, 0, entries * sizeof(uint4), s));  // epoch 0 = empty
    t.ptr = t.own.ptr;
    t.epoch0 = 0;
    return;
  }
  if (ix->ep_entries < entries) {
    if (ix->ep_table) {
      FMG_CK(cudaStreamSynchronize(s));  // no launch of this index may still use it (we hold the lease)
      dfree(ix->ep_table);
      ix->ep_table = nullptr;
      ix->ep_entries = 0;
    }
    FMG_CK(dmalloc(&ix->ep_table, entries * sizeof(uint4)));
    ix->ep_entries = entries;
    ix->ep_next = 0xFFFFFFFFull;  // forces the zeroing below
  }
  if (ix->ep_next + epochs >= 0xFFFFFFFFull) {
    FMG_CK(cudaMemsetAsync(ix->ep_table, 0, ix->ep_entries * sizeof(uint4), s));
    ix->ep_next = 0;
  }
  t.ptr = ix->ep_table;
  t.epoch0 = uint32_t(ix->ep_next);
  ix->ep_next += epochs;
  t.lease = std::move(lk);
}

// z = 1 through k_spine / k_chain; false when a queue overflowed (the caller
// then runs the DFS engine, which has no such limit).  Fills res on success.
// Raw (pattern, k, l, used) results -> the CSR result set of `res`:
// counting sort by pattern, per-pattern sort by (k, l), keep the smallest
// `used` per interval (search.py:127-134, 153-159).
void z1_collect(Z1Raw* raws, uint64_t n_raw, uint64_t count, cudaStream_t s, unsigned long long* steps,
                fmg_matches* res) {
  // group raw results by pattern (counting sort), sort each segment by (k, l)
  DevBuf<uint32_t> per_q(count, s);
  DevBuf<uint64_t> seg(count + 1, s), cursor(count, s), c64(count, s);
  FMG_CK(cudaMemsetAsync(per_q.ptr, 0, count * 4, s));
  FMG_CK(cudaMemsetAsync(seg.ptr, 0, 8, s));
  if (n_raw) k_z1_hist<<<unsigned((n_raw + 255) / 256), 256, 0, s>>>(raws, n_raw, per_q.ptr);
  k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  size_t tb = 0;
  FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, c64.ptr, seg.ptr + 1, count, s));
  DevBuf<uint8_t> tmp(tb, s);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, seg.ptr + 1, count, s));
  FMG_CK(cudaMemcpyAsync(cursor.ptr, seg.ptr, count * 8, cudaMemcpyDeviceToDevice, s));
  const uint64_t nr = std::max<uint64_t>(n_raw, 1);
  DevBuf<uint64_t> keys(nr, s), keys2(nr, s);
  DevBuf<uint8_t> used(nr, s), used2(nr, s);
  if (n_raw) {
    k_z1_scatter<<<unsigned((n_raw + 255) / 256), 256, 0, s>>>(raws, n_raw, cursor.ptr, keys.ptr, used.ptr);
    FMG_REQUIRE(n_raw < (1ull << 31), "too many inexact results for one call");
    size_t sb = 0;
    FMG_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, keys.ptr, keys2.ptr, used.ptr, used2.ptr, int(n_raw),
                                               int(count), seg.ptr, seg.ptr + 1, s));
    DevBuf<uint8_t> stmp(sb, s);
    FMG_CK(cub::DeviceSegmentedSort::SortPairs(stmp.ptr, sb, keys.ptr, keys2.ptr, used.ptr, used2.ptr, int(n_raw),
                                               int(count), seg.ptr, seg.ptr + 1, s));
  }
  k_z1_unique_count<<<unsigned((count + 255) / 256), 256, 0, s>>>(keys2.ptr, used2.ptr, seg.ptr, count, per_q.ptr);
  k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, res->row_off + 1, count, s));
  uint64_t total = 0;
  FMG_CK(cudaMemcpyAsync(&total, res->row_off + count, 8, cudaMemcpyDeviceToHost, s));
  unsigned long long st[2] = {0, 0};
  FMG_CK(cudaMemcpyAsync(st, steps, sizeof(st), cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  res->total = total;
  res->steps = st[0];
  res->lines = st[1];
  FMG_CK(amalloc(reinterpret_cast<void**>(&res->k), std::max<uint64_t>(total, 1) * 4, s));
  FMG_CK(amalloc(reinterpret_cast<void**>(&res->l), std::max<uint64_t>(total, 1) * 4, s));
  FMG_CK(amalloc(reinterpret_cast<void**>(&res->diffs), std::max<uint64_t>(total, 1), s));
  k_z1_unique_write<<<unsigned((count + 255) / 256), 256, 0, s>>>(keys2.ptr, used2.ptr, seg.ptr, res->row_off,
                                                                  count, res->k, res->l, res->diffs);
  FMG_CK(cudaGetLastError());
}

bool run_z1(const fmg_index* ix, const CodePatterns& cp, uint64_t count, uint64_t m, cudaStream_t s,
            unsigned long long* steps, fmg_matches* res) {
  static const bool trace = std::getenv("FMG_TRACE") != nullptr;
  cudaEvent_t ev[4] = {};
  if (trace)
    for (auto& e : ev) cudaEventCreate(&e);
  if (trace) cudaEventRecord(ev[0], s);
  const size_t free_b = available_bytes(ix->device);
  // worst case 8 continuations per spine node and m + 1 spine nodes; in
  // practice far fewer, so cap by memory and detect overflow
  const uint64_t worst = count * 8 * (m + 1);
  const uint64_t budget_entries = std::max<uint64_t>(1u << 20, free_b / 4 / sizeof(Z1Node));
  const uint64_t node_cap = std::min<uint64_t>(worst, budget_entries);
  const uint64_t raw_cap = std::min<uint64_t>(worst + count, budget_entries / 2);
  DevBuf<Z1Node> nodes(node_cap, s);
  DevBuf<Z1Raw> raws(raw_cap, s);
  DevBuf<unsigned long long> ctr(2, s);
  FMG_CK(cudaMemsetAsync(ctr.ptr, 0, 16, s));
  Z1Queues qu{nodes.ptr, ctr.ptr, node_cap, raws.ptr, ctr.ptr + 1, raw_cap};
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    k_spine<W><<<unsigned((count + 255) / 256), 256, 0, s>>>(ix->view(), cp, count, qu, steps);
  });
  FMG_CK(cudaGetLastError());
  unsigned long long n_nodes = 0;
  FMG_CK(cudaMemcpyAsync(&n_nodes, ctr.ptr, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  if (n_nodes > node_cap) return false;
  if (trace) cudaEventRecord(ev[1], s);
  if (n_nodes) {
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      const unsigned nb = persistent_blocks(ix, (const void*)k_chain<W>, 256, n_nodes);
      k_chain<W><<<nb, 256, 0, s>>>(ix->view(), cp, nodes.ptr, n_nodes, qu, steps);
    });
    FMG_CK(cudaGetLastError());
  }
  unsigned long long n_raw = 0;
  FMG_CK(cudaMemcpyAsync(&n_raw, ctr.ptr + 1, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaStreamSynchronize(s));
  if (n_raw > raw_cap) return false;
  if (trace) cudaEventRecord(ev[2], s);
  z1_collect(raws.ptr, n_raw, count, s, steps, res);
  uint64_t total = res->total;
  FMG_CK(cudaGetLastError());
  if (trace) cudaEventRecord(ev[3], s);
  FMG_CK(cudaStreamSynchronize(s));
  if (trace) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    fprintf(stderr, "[fmg] z1 engine: %llu patterns, spine+queue %.3f ms (%llu continuations), chains %.3f ms, "
            "dedup/sort %.3f ms (%llu raw -> %llu results)\n", (unsigned long long)count, a, n_nodes, b, c,
            n_raw, (unsigned long long)total);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  return true;
}

// The level-synchronous bidirectional z = 1 engine (kernels_bidir.cuh),
// host-sync-free: patterns in chunks sized so the worst case of 8
// continuations per spine node always fits the node queue; the chain kernel
// reads the queue length from the device counter; results are grouped by
// pattern (counting sort over device-counted raws), sorted and deduplicated
// per pattern inside one kernel, and written to capacity-sized buffers.  The
// call synchronises ONCE, at the end, to learn the result count, the work
// counters and whether the raw buffer overflowed (then the caller falls back
// to the DFS engine, which gives the same results).
bool run_z1b(const fmg_index* ix, const BiIndex& bi, const CodePatterns& cp, uint64_t count, uint64_t m,
             cudaStream_t s, unsigned long long* steps, fmg_matches* res) {
  static const bool trace = std::getenv("FMG_TRACE") != nullptr;
  cudaEvent_t ev[3] = {};
  if (trace)
    for (auto& e : ev) cudaEventCreate(&e);
  if (trace) cudaEventRecord(ev[0], s);
  const size_t free_b = available_bytes(ix->device);
  const uint64_t per = 8 * (m + 1);
  const uint64_t node_budget = std::max<uint64_t>(per, free_b / 4 / sizeof(Z1BNode));
  const uint64_t chunk = std::min<uint64_t>(count, std::max<uint64_t>(1, node_budget / per));
  const uint64_t node_cap = chunk * per;
  // raws: 16 B each, plus 2 x 9 B of keys / used and 9 B of results below
  const uint64_t raw_cap = std::min<uint64_t>(count * (per + 17), std::max<uint64_t>(1u << 20, free_b / 8 / 43));
  DevBuf<Z1BNode> nodes(node_cap, s);
  DevBuf<Z1Raw> raws(raw_cap, s);
  DevBuf<unsigned long long> ctr(2, s);
  FMG_CK(cudaMemsetAsync(ctr.ptr, 0, 16, s));
  Z1BQueues qu{nodes.ptr, ctr.ptr, node_cap, raws.ptr, ctr.ptr + 1, raw_cap};
  for (uint64_t q0 = 0; q0 < count; q0 += chunk) {
    const uint64_t c = std::min<uint64_t>(chunk, count - q0);
    FMG_CK(cudaMemsetAsync(ctr.ptr, 0, 8, s));
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      k_bspine<W><<<unsigned((c + 255) / 256), 256, 0, s>>>(ix->view(), bi, cp, q0, c, qu, steps);
      // one full-residency wave; lanes refill from the queue length on the device
      const unsigned nb = persistent_blocks(ix, (const void*)k_bchain<W>, 256, c * per);
      k_bchain<W><<<nb, 256, 0, s>>>(ix->view(), bi, cp, nodes.ptr, ctr.ptr, qu, steps);
    });
    FMG_CK(cudaGetLastError());
  }
  if (trace) cudaEventRecord(ev[1], s);
  // ---- group by pattern, sort + dedup per pattern, CSR rows ----
  DevBuf<uint32_t> per_q(count, s);
  DevBuf<uint64_t> seg(count + 1, s), cursor(count, s), c64(count, s);
  DevBuf<uint64_t> keys(raw_cap, s);
  DevBuf<uint8_t> used(raw_cap, s);
  FMG_CK(cudaMemsetAsync(per_q.ptr, 0, count * 4, s));
  FMG_CK(cudaMemsetAsync(seg.ptr, 0, 8, s));
  const unsigned gs = unsigned(std::max(1, blocks_per_sm((const void*)k_z1_scatter_dev, 256, 0)) * ix->sms);
  k_z1_hist_dev<<<gs, 256, 0, s>>>(raws.ptr, ctr.ptr + 1, raw_cap, per_q.ptr);
  const unsigned gq = unsigned((count + 255) / 256);
  k_widen_counts<<<gq, 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  size_t tb = 0;
  FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, c64.ptr, seg.ptr + 1, count, s));
  DevBuf<uint8_t> tmp(tb, s);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, seg.ptr + 1, count, s));
  FMG_CK(cudaMemcpyAsync(cursor.ptr, seg.ptr, count * 8, cudaMemcpyDeviceToDevice, s));
  k_z1_scatter_dev<<<gs, 256, 0, s>>>(raws.ptr, ctr.ptr + 1, raw_cap, cursor.ptr, keys.ptr, used.ptr);
  k_z1_sort_unique<<<gq, 256, 0, s>>>(keys.ptr, used.ptr, seg.ptr, count, per_q.ptr);
  k_widen_counts<<<gq, 256, 0, s>>>(count, per_q.ptr, c64.ptr);
  FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, res->row_off + 1, count, s));
  FMG_CK(amalloc(reinterpret_cast<void**>(&res->kl), raw_cap * 8, s));
  FMG_CK(amalloc(reinterpret_cast<void**>(&res->diffs), raw_cap, s));
  k_z1_write_kl<<<gq, 256, 0, s>>>(keys.ptr, used.ptr, seg.ptr, res->row_off, count, res->kl, res->diffs);
  FMG_CK(cudaGetLastError());
  // ---- the one synchronisation: result count, work counters, overflow ----
  struct Info {
    unsigned long long n_raw, total, steps, lines;
  };
  static thread_local Info* info = nullptr;  // pinned, per host thread
  if (!info) FMG_CK(cudaMallocHost(reinterpret_cast<void**>(&info), sizeof(Info)));
  FMG_CK(cudaMemcpyAsync(&info->n_raw, ctr.ptr + 1, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaMemcpyAsync(&info->total, res->row_off + count, 8, cudaMemcpyDeviceToHost, s));
  FMG_CK(cudaMemcpyAsync(&info->steps, steps, 16, cudaMemcpyDeviceToHost, s));
  if (trace) cudaEventRecord(ev[2], s);
  FMG_CK(cudaStreamSynchronize(s));
  if (info->n_raw > raw_cap) {  // overflow: drop these results, the DFS engine redoes the batch
    afree(res->kl, s);
    afree(res->diffs, s);
    res->kl = nullptr;
    res->diffs = nullptr;
    return false;
  }
  res->total = info->total;
  res->steps = info->steps;
  res->lines = info->lines;
  if (trace) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    fprintf(stderr, "[fmg] z1 bidirectional engine: %llu patterns in chunks of %llu, spines+chains %.3f ms, "
            "group/sort/dedup %.3f ms (%llu raw -> %llu results)\n", (unsigned long long)count,
            (unsigned long long)chunk, a, b, info->n_raw, (unsigned long long)res->total);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  return true;
}

// Grows the device's stream-ordered pool once per process to `bytes` of
// reserved memory (one allocation, freed at once; the unlimited release
// threshold keeps it), so the per-call scratch of large searches is carved
// out of already-mapped memory instead of growing the pool mid-run
// (config 3: 30-290 ms stalls in the calls that grew it; config 2 on a
// fresh box: 12-64 ms stalls in the level-synchronous engine's queues).
// FMG_POOL_RESERVE_GB overrides the size (0 disables).
void pool_reserve(int device, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static std::unordered_map<int, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done[device] || guard_mode()) return;
  done[device] = true;
  if (const char* e = std::getenv("FMG_POOL_RESERVE_GB")) bytes = size_t(std::atof(e) * double(size_t(1) << 30));
  if (bytes == 0) return;
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();  // no room: the pool just grows on demand
    return;
  }
  FMG_CK(cudaFreeAsync(p, s));
  FMG_CK(cudaStreamSynchronize(s));
}

// The flat engine's presence filter (kernels_flat.cuh): B = kx + 2 (config 3:
// 18, 8.6 GB per copy), as many copies as fit a third of the available memory
// up to ceil(B / 4) (one group of four window positions per 32-byte sector),
// groups widened when fewer copies fit.  Built once per index from the
// level-kx table.  FMG_FLAT_FILTER=0 disables it, FMG_FLAT_FILTER_NO=n and
// FMG_FLAT_FILTER_D=1..3 (B = kx + D) override the shape (A/B).
FlatFilter flat_filter(const fmg_index* cix, const uint2* tx, uint32_t kx, uint64_t max_len, cudaStream_t s) {
  const bool enabled = [] {  // read per call (tests flip it)
    const char* e = std::getenv("FMG_FLAT_FILTER");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (!enabled || !tx) return {};
  auto* ix = const_cast<fmg_index*>(cix);  // a cache, like the tables
  std::lock_guard<std::mutex> lock(ix->lut_mu);
  if (!ix->flt_tried) {
    int D = 2;
    if (const char* e = std::getenv("FMG_FLAT_FILTER_D")) D = std::min(3, std::max(1, std::atoi(e)));
    const uint32_t B = kx + uint32_t(D);
    if (max_len < B || B > 20) return {};  // nothing (or too little) to filter for these patterns: decide later
    ix->flt_tried = true;
    const uint64_t bytes_per = (uint64_t(1) << (2 * B)) / 8;
    uint32_t NO = (B + 3) / 4;
    if (const char* e = std::getenv("FMG_FLAT_FILTER_NO")) NO = std::min<uint32_t>((B + 1) / 2, std::max(1, std::atoi(e)));
    const size_t room = available_bytes(ix->device) / 3;
    const uint32_t no_min = (B + 14) / 15;  // G <= 15: a variant's bit offset fits 32 bits (k_flat_probe)
    NO = std::max(NO, no_min);
    while (NO > no_min && bytes_per * NO > room) --NO;
    if (bytes_per * NO > room) return {};
    uint32_t* bits = nullptr;
    if (dmalloc(&bits, bytes_per * NO) != cudaSuccess) {
      cudaGetLastError();
      return {};
    }
    FlatFilter f{bits, B, (B + NO - 1) / NO, NO, 0};
    f.rcpG = uint32_t(((uint64_t(1) << 32) + f.G - 1) / f.G);  // G >= 2
    const auto t0 = std::chrono::steady_clock::now();
    FMG_CK(cudaMemsetAsync(bits, 0, bytes_per * NO, s));
    const uint64_t cnt = uint64_t(1) << (2 * kx);
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      const unsigned blocks = unsigned((cnt + 255) / 256);
      if (D == 1) k_flat_filter_build<W, 1><<<blocks, 256, 0, s>>>(ix->view(), tx, cnt, f, bits);
      else if (D == 2) k_flat_filter_build<W, 2><<<blocks, 256, 0, s>>>(ix->view(), tx, cnt, f, bits);
      else k_flat_filter_build<W, 3><<<blocks, 256, 0, s>>>(ix->view(), tx, cnt, f, bits);
    });
    FMG_CK(cudaGetLastError());
    FMG_CK(cudaStreamSynchronize(s));
    if (std::getenv("FMG_TRACE"))
      fprintf(stderr, "[fmg] flat filter: B=%u G=%u copies=%u, %.2f GB, built in %.1f ms\n", f.B, f.G, f.NO,
              double(bytes_per * NO) / 1e9,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    ix->flt_bits = bits;
    ix->flt_B = f.B;
    ix->flt_G = f.G;
    ix->flt_NO = f.NO;
  }
  if (!ix->flt_bits) return {};
  return FlatFilter{ix->flt_bits, ix->flt_B, ix->flt_G, ix->flt_NO,
                    uint32_t(((uint64_t(1) << 32) + ix->flt_G - 1) / ix->flt_G)};
}

// The flat z = 1 engine is the default while the pattern is at most this many
// characters longer than the deepest table level (each extra character is
// one more dependent step for the candidates still alive).
constexpr uint64_t kFlatTail = 6;

// The calling thread's auxiliary streams on `device` for the flat engine's
// chunk pipeline (created once per thread and device, non-blocking).
cudaStream_t flat_stream(int device, int slot) {
  thread_local std::unordered_map<int, std::array<cudaStream_t, 4>> cache;
  auto it = cache.find(device);
  if (it == cache.end()) {
    std::array<cudaStream_t, 4> st{};
    for (auto& x : st) FMG_CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    it = cache.emplace(device, st).first;
  }
  return it->second[size_t(slot)];
}

// Whether a z = 1 batch goes to the flat engine (kernels_flat.cuh), and the
// level-(K + 1) table it gathers from when that is the exact search's table.
// One place for run_inexact and fmg_inexact_wants_reverse.
struct FlatChoice {
  bool use = false;
  const uint2* tx = nullptr;
  uint32_t kx = 0;
};

FlatChoice flat_choice(const fmg_index* ix, uint64_t count, uint64_t max_len, uint32_t z, const PrefixTable& pt,
                       cudaStream_t s) {
  FlatChoice fc;
  const bool force_dfs = std::getenv("FMG_INEXACT_DFS") != nullptr;  // read per call (tests flip it)
  const char* ee = std::getenv("FMG_BIDIR_ENGINE");
  const std::string engine_env(ee ? ee : "");
  uint64_t line_bytes = 0;
  with_words(ix, [&](auto wt) { line_bytes = ix->n_lines * fmg::LineTraits<decltype(wt)::value>::kBytes; });
  if (z == 1 && max_len <= 31 && pt.base && !force_dfs &&
      (engine_env == "flat" || (engine_env.empty() && line_bytes > (uint64_t(64) << 20)))) {
    if (exact_table_level(ix, pt) == pt.k + 1) {
      const KmerTable kt = kmer_table(ix, count, s);
      if (kt.lut && kt.k == pt.k + 1) {
        fc.tx = kt.lut;
        fc.kx = kt.k;
      }
    }
    const uint32_t kmax = fc.tx ? fc.kx : pt.k;
    fc.use = engine_env == "flat" || max_len <= uint64_t(kmax) + kFlatTail;
  }
  return fc;
}

fmg_matches* run_inexact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                         uint64_t max_len, int max_diff, cudaStream_t s, const uint64_t* packed1 = nullptr) {
  FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
  FMG_REQUIRE(max_diff <= 255, "difference budget above 255 is not supported (diffs are stored as u8)");
  FMG_REQUIRE(max_len < 0xFFFF, "pattern longer than 65534 is not supported");
  FMG_REQUIRE(count < 0xFFFFFFFFull, "too many patterns in one call");
  const auto t_entry = std::chrono::steady_clock::now();
  if (count >= (1u << 16)) pool_reserve(ix->device, std::min<size_t>(available_bytes(ix->device) / 4, size_t(32) << 30), s);
  auto* res = new fmg_matches();
  res->device = ix->device;
  res->stream = s;  // the result buffers are pool allocations of this stream: freed on it too
  res->patterns = count;
  try {
    FMG_CK(amalloc(reinterpret_cast<void**>(&res->row_off), (count + 1) * sizeof(uint64_t), s));
    FMG_CK(cudaMemsetAsync(res->row_off, 0, sizeof(uint64_t), s));
    if (count == 0) {
      FMG_CK(cudaStreamSynchronize(s));
      return res;
    }
    const uint32_t z = uint32_t(max_diff);
    const bool short_pat = max_len <= 64;
    const void* kfn = nullptr;
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      kfn = short_pat ? (const void*)k_inexact<true, W> : (const void*)k_inexact<false, W>;
    });
    int smem_optin = 0;
    FMG_CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix->device));

    DevBuf<uint64_t> res_off(count, s);
    DevBuf<uint32_t> res_cnt(count, s);
    DevBuf<uint8_t> res_pass(count, s);
    DevBuf<unsigned long long> counters(6, s);  // total, fail_count, steps, lines, queue cursor, unsorted
    DevBuf<uint32_t> unsorted_list(count, s);
    DevBuf<uint32_t> too_big(1, s);
    FMG_CK(cudaMemsetAsync(too_big.ptr, 0, 4, s));
    bool need_cub_sort = false;
    FMG_CK(cudaMemsetAsync(res_pass.ptr, 0xFF, count, s));
    FMG_CK(cudaMemsetAsync(counters.ptr + 2, 0, 2 * sizeof(unsigned long long), s));
    FMG_CK(cudaMemsetAsync(counters.ptr + 5, 0, sizeof(unsigned long long), s));

    DevBuf<ulonglong2> packed((short_pat && !packed1) ? count : 0, s);
    if (short_pat && !packed1) {
      k_pack_patterns<<<unsigned((count + 255) / 256), 256, 0, s>>>(codes, offsets, count, packed.ptr);
      FMG_CK(cudaGetLastError());
    }
    // shallow DFS nodes step through the prefix table (FMG_INEXACT_LUT=0: off, A/B)
    const bool lut_off = [] {
      const char* e = std::getenv("FMG_INEXACT_LUT");
      return e != nullptr && std::atoi(e) == 0;
    }();
    const PrefixTable pt = lut_off ? PrefixTable{} : prefix_table(ix, count, s);
    DevBuf<uint64_t> dbits(short_pat ? count : 0, s);
    // the flat engine (decided here) runs the lower-bound pass chunk by chunk on its own streams
    const FlatChoice fc = flat_choice(ix, count, max_len, z, pt, s);
    // the lower-bound pass resolves each present run's first Kt characters
    // with one table gather (absent runs: a binary search over the levels)
    // instead of Kt dependent Occ steps; the level-(K + 1) table joins in
    // when it is the exact search's table
    const uint2* db_tx = nullptr;
    uint32_t db_kx = 0;
    if (short_pat) {
      std::lock_guard<std::mutex> lock(const_cast<fmg_index*>(ix)->lut_mu);
      if (pt.base && ix->lut_x && ix->lut_x_k == pt.k + 1) {
        db_tx = ix->lut_x;
        db_kx = ix->lut_x_k;
      }
    }
    auto launch_dbound = [&](uint64_t c0, uint64_t cn, cudaStream_t sd) {  // patterns c0 .. c0 + cn - 1
      CodePatterns cpd{codes, offsets ? offsets + c0 : nullptr, packed.ptr ? packed.ptr + c0 : nullptr,
                       packed1 ? packed1 + c0 : nullptr, uint32_t(max_len)};
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        k_dbound<W><<<unsigned((cn + 255) / 256), 256, 0, sd>>>(ix->view(), cpd, cn, dbits.ptr + c0,
                                                                 counters.ptr + 2, pt, db_tx, db_kx);
      });
      FMG_CK(cudaGetLastError());
    };
    if (short_pat && !fc.use) launch_dbound(0, count, s);
    // z = 1 on an L2-resident index without a reverse index: the
    // level-synchronous engine (uniform warps).  On HBM-resident indexes the
    // DFS engine wins: its chains start from intervals already in L1/L2, while
    // queued continuations re-fetch pattern, bound and first line from DRAM
    // (tools/prof_c3.py).  With a reverse index attached the bidirectional
    // split engine below beats both (config 2: 9.4 -> 6.4 ms per 1M seeds).
    const bool force_dfs = std::getenv("FMG_INEXACT_DFS") != nullptr;  // read per call (tests flip it)
    const bool has_rev = ix->rev_lines.load(std::memory_order_acquire) != nullptr;
    const std::string engine_env = [] {  // read per call (tests flip it)
      const char* e = std::getenv("FMG_BIDIR_ENGINE");
      return std::string(e ? e : "");
    }();
    const bool bidir_off_env = [] {
      const char* e = std::getenv("FMG_INEXACT_BIDIR");
      return e != nullptr && std::atoi(e) == 0;
    }();
    uint64_t line_bytes = 0;
    with_words(ix, [&](auto wt) { line_bytes = ix->n_lines * fmg::LineTraits<decltype(wt)::value>::kBytes; });
    // z = 1, patterns a few characters longer than the deepest table level,
    // HBM-resident index: the flat engine (kernels_flat.cuh) — every string
    // of the one-edit neighbourhood is one table gather plus at most
    // m + 1 - kmax backward steps, a warp per pattern, no reverse index.
    // Config 3 (m = 19, level 16): 113 -> 32 ms per 14M seeds, profiles/r02_flat.md.
    // FMG_BIDIR_ENGINE=flat forces it (any size, m <= 31), any other value
    // keeps it off.
    const uint2* flat_tx = fc.tx;
    const uint32_t flat_kx = fc.kx;
    const bool use_flat = fc.use;
    if (z == 1 && short_pat && !force_dfs && !use_flat && line_bytes <= (uint64_t(64) << 20) &&
        (!has_rev || bidir_off_env)) {
      CodePatterns cpz{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      if (run_z1(ix, cpz, count, max_len, s, counters.ptr + 2, res)) return res;
      // queues overflowed: fall through to the DFS engine (same results)
    }
    // z = 1 with a reverse index attached: the bidirectional engine for the
    // first pass (FMG_INEXACT_BIDIR=0: off, A/B); retries use the DFS engine.
    const bool bidir_off = [] {
      const char* e = std::getenv("FMG_INEXACT_BIDIR");
      return e != nullptr && std::atoi(e) == 0;
    }();
    BiIndex bi{};
    bool bidir = false;
    if (z == 1 && short_pat && has_rev && pt.base && !bidir_off && !use_flat) {
      bi.rev = ix->view_rev();
      bi.tf = pt;
      bi.tr = prefix_table_rev(ix, count, s);
      for (int d = 0; d < 16; ++d) bi.tail[d] = ix->tail[d];
      bidir = bi.tr.base != nullptr;
      static const bool jump_x = [] {  // FMG_BI_JUMPX=0: case-A jumps stop at level K (A/B)
        const char* e = std::getenv("FMG_BI_JUMPX");
        return e == nullptr || std::atoi(e) != 0;
      }();
      if (bidir && jump_x && exact_table_level(ix, pt) == pt.k + 1) {  // the jumps need exactly level K + 1
        const KmerTable kt = kmer_table(ix, count, s);
        if (kt.lut && kt.k == pt.k + 1) {
          bi.tx = kt.lut;
          bi.kx = kt.k;
        }
      }
    }
    const void* kfn_bi = nullptr;
    with_words(ix, [&](auto wt) { kfn_bi = (const void*)k_inexact_bi<decltype(wt)::value, 0>; });
    // bidirectional forms: "split" (phase-uniform case-A and case-B DFS
    // launches + merge; default for HBM-resident indexes), "sync"
    // (level-synchronous spine + chain kernels; default when the line array
    // is L2-resident: config 2 5.9 -> 3.6 ms per 1M seeds, while on config 3
    // its queued continuations re-fetch from DRAM), "dfs" (both cases per
    // thread); FMG_BIDIR_ENGINE selects.
    const std::string bidir_engine =
        !engine_env.empty() ? engine_env : line_bytes <= (uint64_t(64) << 20) ? "sync" : "split";
    const bool bidir_dfs = bidir_engine == "dfs";
    bool bidir_split = bidir && bidir_engine == "split";
    if (bidir && bidir_engine == "sync") {
      CodePatterns cpz{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      static const bool trace_pre = std::getenv("FMG_TRACE") != nullptr;
      if (trace_pre) {  // host time spent before the engine (packing, bound pass, tables, setup)
        FMG_CK(cudaStreamSynchronize(s));
        fprintf(stderr, "[fmg] pre-engine host time %.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count());
      }
      if (run_z1b(ix, bi, cpz, count, max_len, s, counters.ptr + 2, res)) return res;
      // raw-result buffer overflowed: fall through (same results)
      FMG_CK(cudaMemsetAsync(counters.ptr + 2, 0, 2 * sizeof(unsigned long long), s));
    }
    std::vector<DevBuf<uint2>> pass_kl;
    std::vector<DevBuf<uint8_t>> pass_d;
    DevBuf<uint32_t> lists[2] = {DevBuf<uint32_t>(count, s), DevBuf<uint32_t>(count, s)};
    const uint32_t* list = nullptr;  // pass 0: every pattern
    uint64_t pending = count;
    // R: results per pattern before a retry (per-thread hash table of 2R
    // slots).  cap: results per pass (9 bytes each) before patterns finishing
    // later are retried — sized from free memory so a pass rarely fills it.
    uint32_t R = 256;
    if (const char* e = std::getenv("FMG_INEXACT_R")) {  // A/B: first-pass results per pattern (power of 2)
      const uint32_t r = uint32_t(std::atoi(e));
      if (r >= 16 && (r & (r - 1)) == 0) R = r;
    }
    const size_t free_b = available_bytes(ix->device);
    uint64_t cap = std::max<uint64_t>(count * 16, 1u << 20);
    cap = std::min<uint64_t>(cap, std::max<uint64_t>(1u << 20, free_b / 4 / 9));
    // Stack: depth <= 8(z+1) with the budget-ordered pushes of k_inexact;
    // 9(m+z+1)+2 bounds any visiting order.  Grown on overflow.
    const uint32_t S_max = uint32_t(9 * (max_len + z + 1) + 2);
    // The stack is budget-monotone: at most one budget-z entry (the pending
    // spine child) and at most 9 entries per lower budget level, so 9z + 2
    // slots suffice.  Kept small on purpose: shared memory and L1 share the
    // SM's SRAM, and for HBM-resident indexes the L1 left over is worth 30%
    // (config 3: S = 20 -> 667 ms, S = 10 -> 447 ms per 14M seeds).
    uint32_t S = std::min<uint32_t>(std::min<uint32_t>(S_max, 9 * z + 2),
                                    uint32_t(size_t(smem_optin) / (12 * 32)) - 1);
    if (const char* e = std::getenv("FMG_STACK_S")) S = std::max<uint32_t>(2, uint32_t(std::atoi(e)));  // A/B
    int first_pass = 0;
    DevBuf<uint32_t> retry_list;
    if (use_flat) {
      // ---- pass 0 = the flat engine; patterns that do not fit this pass's
      // result buffer are retried by the DFS engine below ----
      // the filter's traversal starts from the deepest table level the engine gathers from
      const FlatFilter flt = flat_tx ? flat_filter(ix, flat_tx, flat_kx, max_len, s)
                                     : flat_filter(ix, pt.base + PrefixTable::off64(pt.k), pt.k, max_len, s);
      // with the filter the output rows are the survivor segments (and the
      // slab tails between them), not the results alone: room for 24 per pattern
      if (flt.bits)
        cap = std::min<uint64_t>(std::max<uint64_t>(cap, count * 24), std::max<uint64_t>(1u << 20, free_b / 4 / 9));
      pass_kl.emplace_back(cap, s);
      pass_d.emplace_back(cap, s);
      FMG_CK(cudaMemsetAsync(counters.ptr, 0, 2 * sizeof(unsigned long long), s));
      FMG_CK(cudaMemsetAsync(counters.ptr + 4, 0, sizeof(unsigned long long), s));
      InexactOut o{};
      o.kl = pass_kl.back().ptr;
      o.diffs = pass_d.back().ptr;
      o.total = counters.ptr;
      o.cap = cap;
      o.res_off = res_off.ptr;
      o.res_cnt = res_cnt.ptr;
      o.res_pass = res_pass.ptr;
      o.pass = 0;
      o.fail_list = lists[0].ptr;
      o.fail_count = counters.ptr + 1;
      o.steps = counters.ptr + 2;
      o.next = counters.ptr + 4;
      o.unsorted = counters.ptr + 5;
      o.unsorted_list = unsorted_list.ptr;
      CodePatterns cp{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      // survivor queue sized for EVERY candidate of a chunk of patterns (no
      // overflow path to get wrong): 24 bytes per entry, an eighth of the
      // available memory, patterns in chunks of cap / (8 m + 1)
      const uint64_t max_cand = 8 * max_len + 1;
      // Survivor queue: with the filter a pattern keeps ~11 of its 8m + 1
      // candidates (config 3), so a chunk is sized for 48 per pattern on
      // average, and always for one pattern's worth; a chunk whose patterns
      // keep more than that overflows into the retry list (DFS engine).
      // Without a filter every candidate survives the probe.  At most 2^25
      // entries (0.75 GB) per stream: large buffers cost more to allocate than
      // the extra chunk launches (12 GB queues: 40-100 ms per call against 44 ms
      // of work), and smaller chunks pipeline better across the streams.
      uint64_t per_pat = flt.bits ? std::min<uint64_t>(max_cand, 48) : max_cand;
      if (const char* e = std::getenv("FMG_FLAT_PER_PAT")) per_pat = std::max(1, std::atoi(e));  // tests: force overflow
      uint64_t q_cap_max = uint64_t(1) << 25;
      if (const char* e = std::getenv("FMG_FLAT_QCAP_LOG2")) q_cap_max = uint64_t(1) << std::min(30, std::max(16, std::atoi(e)));  // A/B
      const uint64_t q_cap = std::max<uint64_t>(
          std::getenv("FMG_FLAT_PER_PAT") ? per_pat : max_cand * 64,
          std::min<uint64_t>(count * per_pat, std::min<uint64_t>(q_cap_max, free_b / 8 / 24)));
      const uint64_t chunk = std::max<uint64_t>(1, q_cap / per_pat);
      // Chunks are pipelined over up to four streams, each with its own
      // queue: the probe is SM-issue-bound, the extend kernel DRAM-request-
      // bound and the collect kernel shared-memory-bound, so chunk i + 1's
      // probe runs under chunk i's extend instead of after it.  Grids are
      // sized so blocks of different kernels fit an SM together.
      // FMG_FLAT_STREAMS=1..4 (1: everything on the caller's stream) and
      // FMG_FLAT_BPS=p,e,c (resident blocks per SM of each kernel) are A/B hooks.
      const uint64_t n_chunks = (count + chunk - 1) / chunk;
      int nstr = 4;
      if (const char* e = std::getenv("FMG_FLAT_STREAMS")) nstr = std::min(4, std::max(1, std::atoi(e)));
      nstr = int(std::min<uint64_t>(uint64_t(nstr), n_chunks));
      std::vector<DevBuf<FlatSurvivor>> surv;
      std::vector<DevBuf<uint2>> raw;
      for (int j = 0; j < nstr; ++j) {
        surv.emplace_back(q_cap, s);
        raw.emplace_back(q_cap, s);
      }
      DevBuf<uint64_t> seg_base(count, s);
      DevBuf<uint32_t> seg_cnt(count, s);
      DevBuf<unsigned long long> n_surv(size_t(nstr), s);
      DevBuf<unsigned long long> rows_base(n_chunks + 1, s);
      FMG_CK(cudaMemsetAsync(rows_base.ptr, 0, sizeof(unsigned long long), s));
      const int nrs = int((3 * max_len + 1 + 31) / 32);  // rounds of 32 slots, 1..3 (m <= 31)
      static const bool trace_flat = std::getenv("FMG_TRACE") != nullptr;
      cudaEvent_t fe[2] = {};
      if (trace_flat) {
        FMG_CK(cudaStreamSynchronize(s));
        fprintf(stderr, "[fmg] flat pre-engine host time %.3f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count());
        for (auto& e : fe) cudaEventCreate(&e);
        cudaEventRecord(fe[0], s);
      }
      const bool fixed_m = packed1 != nullptr;
      const void* kp = fixed_m ? (nrs == 1 ? (const void*)k_flat_probe<1, true> : nrs == 2 ? (const void*)k_flat_probe<2, true>
                                                                                           : (const void*)k_flat_probe<3, true>)
                               : (nrs == 1 ? (const void*)k_flat_probe<1, false> : nrs == 2 ? (const void*)k_flat_probe<2, false>
                                                                                            : (const void*)k_flat_probe<3, false>);
      // with the filter a pattern's survivor segment is also its output
      // reservation (no atomics); without one the rows are reserved exactly
      const bool seg_rows = flt.bits != nullptr;
      int occ_p = std::max(1, blocks_per_sm(kp, 256, 0));
      int occ_c = std::max(1, blocks_per_sm(seg_rows ? (const void*)k_flat_collect<true>
                                                     : (const void*)k_flat_collect<false>, 256, 0));
      int occ_e = 1;
      with_words(ix, [&](auto wt) {
        occ_e = std::max(1, blocks_per_sm((const void*)k_flat_extend<decltype(wt)::value>, 256, 0));
      });
      // (grids capped at 2-3 blocks per SM so that kernels of different chunks
      // share every SM measured slower than full grids taking turns: 25.3 vs
      // 22.5 ms per 14M config-3 seeds, profiles/r02_ab_flat_streams.log)
      if (const char* e = std::getenv("FMG_FLAT_BPS")) {
        int lp = 99, le = 99, lc = 99;
        std::sscanf(e, "%d,%d,%d", &lp, &le, &lc);
        occ_p = std::min(occ_p, std::max(1, lp));
        occ_e = std::min(occ_e, std::max(1, le));
        occ_c = std::min(occ_c, std::max(1, lc));
      }
      const int bp = occ_p * ix->sms, be = occ_e * ix->sms, bc = occ_c * ix->sms;
      // streams and events of this call (nstr == 1: the caller's stream, no events)
      std::vector<cudaStream_t> st(size_t(nstr), s);
      struct Events {  // destroyed on every way out of the call
        std::vector<cudaEvent_t> v;
        cudaEvent_t make() {
          cudaEvent_t e = nullptr;
          FMG_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          v.push_back(e);
          return e;
        }
        ~Events() {
          for (cudaEvent_t e : v) cudaEventDestroy(e);
        }
      } events;
      std::vector<cudaEvent_t> ev_adv(nstr > 1 ? n_chunks : 0), ev_join(nstr > 1 ? size_t(nstr) : 0);
      cudaEvent_t ev_fork = nullptr;
      if (nstr > 1) {
        for (int j = 0; j < nstr; ++j) st[size_t(j)] = flat_stream(ix->device, j);
        ev_fork = events.make();
        for (auto& e : ev_adv) e = events.make();
        for (auto& e : ev_join) e = events.make();
        FMG_CK(cudaEventRecord(ev_fork, s));
        for (int j = 0; j < nstr; ++j) FMG_CK(cudaStreamWaitEvent(st[size_t(j)], ev_fork, 0));
      }
      uint64_t ci = 0;
      try {
      for (uint64_t c0 = 0; c0 < count; c0 += chunk, ++ci) {
        const uint64_t cn = std::min<uint64_t>(chunk, count - c0);
        const size_t j = size_t(ci % uint64_t(nstr));
        cudaStream_t sj = st[j];
        FlatQueues fq{surv[j].ptr, raw[j].ptr, n_surv.ptr + j, q_cap, seg_base.ptr, seg_cnt.ptr};
        FMG_CK(cudaMemsetAsync(fq.n_surv, 0, sizeof(unsigned long long), sj));
        launch_dbound(c0, cn, sj);
        const unsigned gp = unsigned(std::min<uint64_t>(uint64_t(bp), (cn + 7) / 8));  // 8 warps per block
        if (fixed_m) {
          if (nrs == 1) k_flat_probe<1, true><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
          else if (nrs == 2) k_flat_probe<2, true><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
          else k_flat_probe<3, true><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
        } else {
          if (nrs == 1) k_flat_probe<1, false><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
          else if (nrs == 2) k_flat_probe<2, false><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
          else k_flat_probe<3, false><<<gp, 256, 0, sj>>>(cp, nullptr, c0, cn, flt, fq, o);
        }
        with_words(ix, [&](auto wt) {
          constexpr int W = decltype(wt)::value;
          k_flat_extend<W><<<unsigned(be), 256, 0, sj>>>(ix->view(), pt, flat_tx, flat_kx, fq, counters.ptr + 2);
        });
        const unsigned gc = unsigned(std::min<uint64_t>(uint64_t(bc), (cn + 7) / 8));  // 8 warps per block
        if (seg_rows) {
          // rows of this chunk start where the previous chunk's end (another stream's advance)
          if (nstr > 1 && ci > 0) FMG_CK(cudaStreamWaitEvent(sj, ev_adv[ci - 1], 0));
          k_flat_advance<<<1, 1, 0, sj>>>(rows_base.ptr + ci, fq.n_surv, q_cap, counters.ptr);
          if (nstr > 1) FMG_CK(cudaEventRecord(ev_adv[ci], sj));
          k_flat_collect<true><<<gc, 256, 0, sj>>>(nullptr, c0, cn, fq, o, rows_base.ptr + ci);
        } else {
          k_flat_collect<false><<<gc, 256, 0, sj>>>(nullptr, c0, cn, fq, o, nullptr);
        }
        res->launches += seg_rows ? 5 : 4;
        FMG_CK(cudaGetLastError());
      }
      if (nstr > 1) {
        for (int j = 0; j < nstr; ++j) {
          FMG_CK(cudaEventRecord(ev_join[size_t(j)], st[size_t(j)]));
          FMG_CK(cudaStreamWaitEvent(s, ev_join[size_t(j)], 0));
        }
      }
      } catch (...) {  // nothing of this call may still run on the auxiliary streams when its buffers go
        for (cudaStream_t x : st) cudaStreamSynchronize(x);
        throw;
      }
      unsigned long long host_ctr[2];
      FMG_CK(cudaMemcpyAsync(host_ctr, counters.ptr, sizeof(host_ctr), cudaMemcpyDeviceToHost, s));
      if (trace_flat) cudaEventRecord(fe[1], s);
      FMG_CK(cudaStreamSynchronize(s));
      if (trace_flat) {
        float ms = 0;
        cudaEventElapsedTime(&ms, fe[0], fe[1]);
        fprintf(stderr, "[fmg] flat z=1 engine: %llu patterns in chunks of %llu on %d stream(s) (probe %d rounds x %d "
                "blocks, extend %d blocks, collect %d blocks; filter B=%u x %u copies): %.3f ms, %llu rows, %llu retried\n",
                (unsigned long long)count, (unsigned long long)chunk, nstr, nrs, bp, be, bc, flt.B, flt.NO, ms,
                host_ctr[0], host_ctr[1]);
        for (auto& e : fe) cudaEventDestroy(e);
      }

      list = lists[0].ptr;
      pending = host_ctr[1];
      first_pass = 1;
      if (pending > 0) cap = std::max<uint64_t>(cap, std::min<uint64_t>(pending * 256, 1ull << 31));
    }
    if (bidir_split) {
      // ---- pass 0 = case-A launch + case-B launch + merge (kernels_bidir.cuh) ----
      const uint32_t Sp = 9;  // z = 1: one budget-1 node's children at a time
      const int nt = 128;
      // stack entries: 12 bytes for case A (one interval), 20 for case B
      const size_t smemA = size_t(Sp + 1) * 12 * nt, smem = size_t(Sp + 1) * 20 * nt;
      FMG_REQUIRE(smem <= size_t(smem_optin), "inexact search stack does not fit in shared memory");
      const void* kA = nullptr;
      const void* kB = nullptr;
      static const bool one_word_ok = [] {  // FMG_BI_ONEWORD=0: the two-word kernels (A/B)
        const char* e = std::getenv("FMG_BI_ONEWORD");
        return e == nullptr || std::atoi(e) != 0;
      }();
      const bool one_word = one_word_ok && max_len <= 32;  // patterns in one 64-bit word: the kOne kernels
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        kA = one_word ? (const void*)k_inexact_bi<W, 1, true> : (const void*)k_inexact_bi<W, 1, false>;
        kB = (const void*)k_inexact_bi<W, 3, false>;  // (kOne for case B spills at 72 registers: 83 -> 98 ms)
      });
      FMG_CK(cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smemA)));
      FMG_CK(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int per_sm = 0;
      int per_sm_b = 0;
      FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kA, nt, smemA));
      FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, kB, nt, smem));
      per_sm = std::max(std::max(per_sm, per_sm_b), 1);  // T sized for the more resident of the two
      const uint64_t per_thread = uint64_t(R) * (2 * 16 + 4);
      uint64_t T = uint64_t(per_sm) * ix->sms * nt;
      T = std::min<uint64_t>(T, std::max<uint64_t>(nt, std::max<uint64_t>(2ull << 30, free_b / 8) / per_thread));
      T = std::min<uint64_t>(T, ((count + nt - 1) / nt) * nt);
      T = std::max<uint64_t>(nt, (T / nt) * nt);
      EpochTable table;
      lease_epoch_table(const_cast<fmg_index*>(ix), uint64_t(2 * R) * T, 2 * (count + 1), s, table);
      DevBuf<uint32_t> slots(uint64_t(R) * T, s);
      InexactScratch sc{};
      sc.table = table.ptr;
      sc.slots = slots.ptr;
      sc.S = Sp;
      sc.R = R;
      sc.Mmax = uint32_t(max_len);
      sc.T = T;
      const uint64_t cap_h = std::max<uint64_t>(1u << 20, cap / 2);
      DevBuf<uint2> klh[2] = {DevBuf<uint2>(cap_h, s), DevBuf<uint2>(cap_h, s)};
      DevBuf<uint8_t> dh[2] = {DevBuf<uint8_t>(cap_h, s), DevBuf<uint8_t>(cap_h, s)};
      DevBuf<uint64_t> offh[2] = {DevBuf<uint64_t>(count, s), DevBuf<uint64_t>(count, s)};
      DevBuf<uint32_t> cnth[2] = {DevBuf<uint32_t>(count, s), DevBuf<uint32_t>(count, s)};
      DevBuf<uint8_t> passh(count, s);
      CodePatterns cp{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      bool too_big_any = false;
      static const bool trace_split = std::getenv("FMG_TRACE") != nullptr;
      cudaEvent_t sev[6] = {};
      if (trace_split)
        for (auto& e : sev) cudaEventCreate(&e);
      unsigned long long n_unsorted[2] = {0, 0};
      for (int half = 0; half < 2; ++half) {
        if (trace_split) cudaEventRecord(sev[2 * half], s);
        sc.epoch0 = table.epoch0 + uint32_t(half) * uint32_t(count + 1);  // each half its own epochs
        FMG_CK(cudaMemsetAsync(counters.ptr, 0, 2 * sizeof(unsigned long long), s));
        FMG_CK(cudaMemsetAsync(counters.ptr + 4, 0, 2 * sizeof(unsigned long long), s));
        InexactOut o{};
        o.kl = klh[half].ptr;
        o.diffs = dh[half].ptr;
        o.total = counters.ptr;
        o.cap = cap_h;
        o.res_off = offh[half].ptr;
        o.res_cnt = cnth[half].ptr;
        o.res_pass = passh.ptr;
        o.pass = 0;
        o.fail_list = lists[0].ptr;
        o.fail_count = counters.ptr + 1;
        o.steps = counters.ptr + 2;
        o.next = counters.ptr + 4;
        o.unsorted = counters.ptr + 5;
        o.unsorted_list = unsorted_list.ptr;
        with_words(ix, [&](auto wt) {
          constexpr int W = decltype(wt)::value;
          if (half == 0 && one_word)
            k_inexact_bi<W, 1, true><<<unsigned(T / nt), nt, smemA, s>>>(ix->view(), bi, cp, nullptr, count, sc, o);
          else if (half == 0)
            k_inexact_bi<W, 1, false><<<unsigned(T / nt), nt, smemA, s>>>(ix->view(), bi, cp, nullptr, count, sc, o);
          else
            k_inexact_bi<W, 3, false><<<unsigned(T / nt), nt, smem, s>>>(ix->view(), bi, cp, nullptr, count, sc, o);
        });
        FMG_CK(cudaGetLastError());
        unsigned long long host_ctr[6];
        FMG_CK(cudaMemcpyAsync(host_ctr, counters.ptr, sizeof(host_ctr), cudaMemcpyDeviceToHost, s));
        if (trace_split) cudaEventRecord(sev[2 * half + 1], s);
        FMG_CK(cudaStreamSynchronize(s));
        n_unsorted[half] = host_ctr[5];
        if (host_ctr[5] > 0) {  // sort this half's large result sets in place
          k_sort_segments<<<unsigned(host_ctr[5]), 256, 0, s>>>(unsorted_list.ptr, offh[half].ptr, cnth[half].ptr,
                                                                klh[half].ptr, dh[half].ptr, too_big.ptr);
          FMG_CK(cudaGetLastError());
          uint32_t tb_flag = 0;
          FMG_CK(cudaMemcpyAsync(&tb_flag, too_big.ptr, 4, cudaMemcpyDeviceToHost, s));
          FMG_CK(cudaStreamSynchronize(s));
          too_big_any = too_big_any || tb_flag;
        }
      }
      if (too_big_any) {
        // a half-list was too long to sort in place, so the merge would be
        // wrong: redo every pattern with the one-directional DFS engine
        bidir_split = false;
        bidir = false;
        FMG_CK(cudaMemsetAsync(too_big.ptr, 0, 4, s));
        FMG_CK(cudaMemsetAsync(res_pass.ptr, 0xFF, count, s));
      } else {
        DevBuf<uint64_t> c64(count, s), moff(count + 1, s);
        DevBuf<unsigned long long> nret(1, s);
        retry_list = DevBuf<uint32_t>(count, s);
        FMG_CK(cudaMemsetAsync(nret.ptr, 0, 8, s));
        FMG_CK(cudaMemsetAsync(moff.ptr, 0, 8, s));
        const unsigned gb = unsigned((count + 255) / 256);
        k_merge_ab<<<gb, 256, 0, s>>>(count, offh[0].ptr, cnth[0].ptr, klh[0].ptr, dh[0].ptr, offh[1].ptr,
                                      cnth[1].ptr, klh[1].ptr, dh[1].ptr, false, c64.ptr, nullptr, nullptr, nullptr,
                                      nullptr, nullptr, nullptr, nullptr, nullptr);
        size_t tb = 0;
        FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, c64.ptr, moff.ptr + 1, count, s));
        DevBuf<uint8_t> tmp(tb, s);
        FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tb, c64.ptr, moff.ptr + 1, count, s));
        uint64_t mtotal = 0;
        FMG_CK(cudaMemcpyAsync(&mtotal, moff.ptr + count, 8, cudaMemcpyDeviceToHost, s));
        FMG_CK(cudaStreamSynchronize(s));
        pass_kl.emplace_back(std::max<uint64_t>(mtotal, 1), s);
        pass_d.emplace_back(std::max<uint64_t>(mtotal, 1), s);
        k_merge_ab<<<gb, 256, 0, s>>>(count, offh[0].ptr, cnth[0].ptr, klh[0].ptr, dh[0].ptr, offh[1].ptr,
                                      cnth[1].ptr, klh[1].ptr, dh[1].ptr, true, nullptr, moff.ptr,
                                      pass_kl.back().ptr, pass_d.back().ptr, res_cnt.ptr, res_off.ptr, res_pass.ptr,
                                      retry_list.ptr, nret.ptr);
        FMG_CK(cudaGetLastError());
        unsigned long long n_retry = 0;
        FMG_CK(cudaMemcpyAsync(&n_retry, nret.ptr, 8, cudaMemcpyDeviceToHost, s));
        FMG_CK(cudaStreamSynchronize(s));
        list = retry_list.ptr;
        pending = n_retry;
        first_pass = 1;
        if (trace_split) {
          cudaEventRecord(sev[5], s);
          cudaEventSynchronize(sev[5]);
          float ta = 0, tsa = 0, tb = 0, tm = 0;
          cudaEventElapsedTime(&ta, sev[0], sev[1]);
          cudaEventElapsedTime(&tsa, sev[1], sev[2]);
          cudaEventElapsedTime(&tb, sev[2], sev[3]);
          cudaEventElapsedTime(&tm, sev[3], sev[5]);
          fprintf(stderr, "[fmg] bidirectional split: case A %.3f ms (%llu > S sorted, %.3f ms), case B %.3f ms "
                  "(%llu > S), B sort + merge %.3f ms, %llu merged results, %llu retried\n", ta, n_unsorted[0], tsa,
                  tb, n_unsorted[1], tm, (unsigned long long)mtotal, n_retry);
        }
      }
    }
    for (int pass = first_pass; pending > 0; ++pass) {
      FMG_REQUIRE(pass < 250, "inexact search did not converge");
      const bool use_bi = bidir && !bidir_split && pass == 0;
      const uint32_t Sp = use_bi ? 9u : S;  // z = 1: one budget-1 node's children at a time
      const size_t ebytes = use_bi ? 20 : 12;
      const void* kf = use_bi ? kfn_bi : kfn;
      int nt = 128;
      while (nt > 32 && size_t(Sp) * ebytes * nt > size_t(96) << 10) nt /= 2;
      const size_t smem = size_t(Sp + 1) * ebytes * nt;  // + the push dump slot
      FMG_REQUIRE(smem <= size_t(smem_optin), "inexact search stack does not fit in shared memory");
      FMG_CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int per_sm = 0;
      FMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, nt, smem));
      per_sm = std::max(per_sm, 1);
      // threads: full residency, bounded by a scratch budget of ~2 GiB
      const uint64_t per_thread = uint64_t(R) * (2 * 16 + 4) + (short_pat ? 0 : max_len);
      uint64_t T = uint64_t(per_sm) * ix->sms * nt;
      T = std::min<uint64_t>(T, std::max<uint64_t>(nt, std::max<uint64_t>(2ull << 30, free_b / 8) / per_thread));
      T = std::min<uint64_t>(T, ((pending + nt - 1) / nt) * nt);
      T = std::max<uint64_t>(nt, (T / nt) * nt);
      InexactScratch sc{};
      EpochTable table;
      lease_epoch_table(const_cast<fmg_index*>(ix), uint64_t(2 * R) * T, pending + 1, s, table);
      DevBuf<uint32_t> slots(uint64_t(R) * T, s);
      DevBuf<uint8_t> dl(short_pat ? 0 : max_len * T, s);
      sc.table = table.ptr;
      sc.epoch0 = table.epoch0;
      sc.slots = slots.ptr;
      sc.dlb = dl.ptr;
      sc.S = Sp;
      sc.R = R;
      sc.Mmax = uint32_t(max_len);
      sc.T = T;
      pass_kl.emplace_back(cap, s);
      pass_d.emplace_back(cap, s);
      FMG_CK(cudaMemsetAsync(counters.ptr, 0, 2 * sizeof(unsigned long long), s));
      FMG_CK(cudaMemsetAsync(counters.ptr + 4, 0, sizeof(unsigned long long), s));
      InexactOut o{};
      o.kl = pass_kl.back().ptr;
      o.diffs = pass_d.back().ptr;
      o.total = counters.ptr;
      o.cap = cap;
      o.res_off = res_off.ptr;
      o.res_cnt = res_cnt.ptr;
      o.res_pass = res_pass.ptr;
      o.pass = uint8_t(pass);
      o.fail_list = lists[pass & 1].ptr;
      o.fail_count = counters.ptr + 1;
      o.steps = counters.ptr + 2;
      o.next = counters.ptr + 4;
      o.unsorted = counters.ptr + 5;
      o.unsorted_list = unsorted_list.ptr;
      FMG_CK(cudaMemsetAsync(counters.ptr + 5, 0, sizeof(unsigned long long), s));
      const unsigned blocks = unsigned(T / nt);
      CodePatterns cp{codes, offsets, packed.ptr, packed1, uint32_t(max_len), dbits.ptr};
      static const bool trace = std::getenv("FMG_TRACE") != nullptr;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (trace) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, s);
      }
      with_words(ix, [&](auto wt) {
        constexpr int W = decltype(wt)::value;
        if (use_bi)
          k_inexact_bi<W, 0><<<blocks, nt, smem, s>>>(ix->view(), bi, cp, list, pending, sc, o);
        else if (short_pat)
          k_inexact<true, W><<<blocks, nt, smem, s>>>(ix->view(), cp, list, pending, z, sc, o, pt);
        else
          k_inexact<false, W><<<blocks, nt, smem, s>>>(ix->view(), cp, list, pending, z, sc, o, pt);
      });
      FMG_CK(cudaGetLastError());
      unsigned long long host_ctr[6];
      FMG_CK(cudaMemcpyAsync(host_ctr, counters.ptr, sizeof(host_ctr), cudaMemcpyDeviceToHost, s));
      FMG_CK(cudaStreamSynchronize(s));
      const uint64_t failed = host_ctr[1];
      if (host_ctr[5] > 0) {  // sort this pass's large result sets in place
        k_sort_segments<<<unsigned(host_ctr[5]), 256, 0, s>>>(unsorted_list.ptr, res_off.ptr, res_cnt.ptr,
                                                              pass_kl.back().ptr, pass_d.back().ptr, too_big.ptr);
        FMG_CK(cudaGetLastError());
        uint32_t tb_flag = 0;
        FMG_CK(cudaMemcpyAsync(&tb_flag, too_big.ptr, 4, cudaMemcpyDeviceToHost, s));
        FMG_CK(cudaStreamSynchronize(s));
        if (tb_flag) need_cub_sort = true;
      }
      if (trace) {
        cudaEventRecord(ev1, s);
        cudaEventSynchronize(ev1);
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        unsigned long long st = 0;
        cudaMemcpy(&st, counters.ptr + 2, 8, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[fmg] inexact pass %d: %llu patterns, T=%llu nt=%d S=%u R=%u smem=%zu per_sm=%d: %.3f ms, "
                "%llu failed, %llu steps so far\n", pass, (unsigned long long)pending, (unsigned long long)T, nt, S,
                R, smem, per_sm, ms, (unsigned long long)failed, st);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
      }
      list = lists[pass & 1].ptr;
      if (failed > 0) {
        // grow whichever capacity might have been the cause; the DFS stack
        // is capped at what shared memory holds at 32 threads per block
        const uint32_t S_fit = uint32_t(size_t(smem_optin) / (12 * 32)) - 1;
        if (R == (1u << 22) && S >= std::min(S_max, S_fit))
          throw std::invalid_argument(
              "inexact search: a pattern needs a DFS stack deeper than shared memory holds (" +
              std::to_string(S_fit) + " entries) or more than 2^22 results; use a smaller max_diff or "
              "shorter patterns");
        R = std::min<uint32_t>(R * 8, 1u << 22);
        S = std::min<uint32_t>(std::min(S_max, S_fit), S * 2);
        cap = std::max<uint64_t>(cap, std::min<uint64_t>(uint64_t(host_ctr[0]) * 2, 1ull << 31));
        cap = std::max<uint64_t>(cap, failed * uint64_t(R));
        cap = std::min<uint64_t>(cap, 1ull << 31);
      }
      pending = failed;
      // the next pass reads `list` while writing the other list
    }
    static const bool trace_post = std::getenv("FMG_TRACE") != nullptr;
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (trace_post) {
      cudaEventCreate(&pe0);
      cudaEventCreate(&pe1);
      cudaEventRecord(pe0, s);
    }
    // CSR: row_off[q+1] = inclusive sum of counts
    DevBuf<uint64_t> c64(count, s);
    if (res->launches) res->launches += 2 + (packed1 ? 0 : 1);  // k_widen_counts, k_gather_matches (+ k_pack_patterns)
    k_widen_counts<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, res_cnt.ptr, c64.ptr);
    size_t tmp_bytes = 0;
    FMG_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, c64.ptr, res->row_off + 1, count, s));
    DevBuf<uint8_t> tmp(tmp_bytes, s);
    FMG_CK(cub::DeviceScan::InclusiveSum(tmp.ptr, tmp_bytes, c64.ptr, res->row_off + 1, count, s));
    uint64_t total = 0;
    FMG_CK(cudaMemcpyAsync(&total, res->row_off + count, sizeof(total), cudaMemcpyDeviceToHost, s));
    unsigned long long work[2] = {0, 0};
    FMG_CK(cudaMemcpyAsync(work, counters.ptr + 2, sizeof(work), cudaMemcpyDeviceToHost, s));
    FMG_CK(cudaStreamSynchronize(s));
    const bool unsorted = need_cub_sort;
    res->total = total;
    res->steps = work[0];
    res->lines = work[1];
    FMG_CK(amalloc(reinterpret_cast<void**>(&res->k), std::max<uint64_t>(total, 1) * sizeof(uint32_t), s));
    FMG_CK(amalloc(reinterpret_cast<void**>(&res->l), std::max<uint64_t>(total, 1) * sizeof(uint32_t), s));
    FMG_CK(amalloc(reinterpret_cast<void**>(&res->diffs), std::max<uint64_t>(total, 1), s));
    for (size_t p = 0; p < pass_kl.size(); ++p) {
      k_gather_matches<<<unsigned((count + 255) / 256), 256, 0, s>>>(count, res_off.ptr, res_cnt.ptr, res_pass.ptr,
                                                                     uint8_t(p), pass_kl[p].ptr, pass_d[p].ptr,
                                                                     res->row_off, res->k, res->l, res->diffs);
      FMG_CK(cudaGetLastError());
    }
    if (unsorted && total > 0) {
      // a pattern had more than kSortMax results: segmented sort of everything by (k, l)
      FMG_REQUIRE(total < (1ull << 31), "too many inexact results for one call");
      DevBuf<uint64_t> keys(total, s), keys2(total, s);
      DevBuf<uint8_t> d2(total, s);
      k_pack_keys<<<unsigned((total + 255) / 256), 256, 0, s>>>(total, res->k, res->l, keys.ptr);
      size_t sb = 0;
      FMG_CK(cub::DeviceSegmentedSort::SortPairs(nullptr, sb, keys.ptr, keys2.ptr, res->diffs, d2.ptr, int(total),
                                                 int(count), res->row_off, res->row_off + 1, s));
      DevBuf<uint8_t> stmp(sb, s);
      FMG_CK(cub::DeviceSegmentedSort::SortPairs(stmp.ptr, sb, keys.ptr, keys2.ptr, res->diffs, d2.ptr, int(total),
                                                 int(count), res->row_off, res->row_off + 1, s));
      k_unpack_keys<<<unsigned((total + 255) / 256), 256, 0, s>>>(total, keys2.ptr, d2.ptr, res->k, res->l,
                                                                   res->diffs);
      FMG_CK(cudaGetLastError());
    }
    FMG_CK(cudaStreamSynchronize(s));
    if (trace_post) {
      cudaEventRecord(pe1, s);
      cudaEventSynchronize(pe1);
      float ms = 0;
      cudaEventElapsedTime(&ms, pe0, pe1);
      fprintf(stderr, "[fmg] inexact post (CSR, gather, %s): %.3f ms, %llu results; whole call %.3f ms of host time\n",
              unsorted ? "segmented sort" : "no sort", ms, (unsigned long long)total,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count());
      cudaEventDestroy(pe0);
      cudaEventDestroy(pe1);
    }
    return res;
  } catch (...) {
    fmg_matches_free(res);
    throw;
  }
}

// The calling thread's streams on `device` for the host-buffer entry points,
// created on first use and kept (never destroyed: a thread-exit destructor
// could run after the CUDA context is gone).  Reusing them keeps per-call
// overhead to the copies and the kernels — creating and destroying three
// streams per call cost more than a 10,000-pattern search (config 0 e2e) —
// and lets the stream-ordered pool reuse the previous call's blocks on the
// same stream.
cudaStream_t host_stream(int device, int slot) {
  thread_local std::unordered_map<int, std::array<cudaStream_t, 3>> cache;
  auto it = cache.find(device);
  if (it == cache.end()) {
    std::array<cudaStream_t, 3> st{};
    for (auto& x : st) FMG_CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    it = cache.emplace(device, st).first;
  }
  return it->second[slot];
}

// Whether p is page-locked host memory the device can address directly
// (cudaHostAlloc / cudaHostRegister under unified addressing).
bool pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// Chunked host-buffer pipeline: H2D, kernel, D2H per chunk on alternating
// streams so the copy engines overlap each other and the kernel.
template <typename Launch>
void pipeline_host(int device, uint64_t count, uint64_t chunk, size_t in_bytes_per, size_t out_bytes_per,
                   const void* host_in, void* host_out, Launch&& launch) {
  if (count == 0) return;
  constexpr int kMaxSlots = 3;
  const int kSlots = int(std::min<uint64_t>(kMaxSlots, (count + chunk - 1) / chunk));  // slots actually used
  cudaStream_t st[kMaxSlots];
  for (int i = 0; i < kSlots; ++i) st[i] = host_stream(device, i);
  std::vector<void*> din(kSlots, nullptr), dout(kSlots, nullptr);
  try {
    for (int i = 0; i < kSlots; ++i) {
      FMG_CK(amalloc(&din[i], std::max<size_t>(chunk * in_bytes_per, 1), st[i]));
      FMG_CK(amalloc(&dout[i], std::max<size_t>(chunk * out_bytes_per, 1), st[i]));
    }
    uint64_t c = 0;
    for (uint64_t off = 0; off < count; off += chunk, ++c) {
      const int slot = int(c % kSlots);
      const uint64_t len = std::min(chunk, count - off);
      FMG_CK(cudaMemcpyAsync(din[slot], static_cast<const uint8_t*>(host_in) + off * in_bytes_per, len * in_bytes_per,
                             cudaMemcpyHostToDevice, st[slot]));
      launch(din[slot], len, dout[slot], st[slot]);
      FMG_CK(cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + off * out_bytes_per, dout[slot], len * out_bytes_per,
                             cudaMemcpyDeviceToHost, st[slot]));
    }
    for (int i = 0; i < kSlots; ++i) FMG_CK(cudaStreamSynchronize(st[i]));
  } catch (...) {
    for (int i = 0; i < kSlots; ++i) cudaStreamSynchronize(st[i]);
    for (int i = 0; i < kSlots; ++i) {
      if (din[i]) afree(din[i], st[i]);
      if (dout[i]) afree(dout[i], st[i]);
      cudaStreamSynchronize(st[i]);
    }
    throw;
  }
  for (int i = 0; i < kSlots; ++i) {
    afree(din[i], st[i]);
    afree(dout[i], st[i]);
  }
}

}  // namespace

extern "C" {

const char* fmg_last_error(void) { return fmg::g_last_error.c_str(); }

int fmg_device_count(int* count) {
  return fmg::guard([&] {
    FMG_REQUIRE(count != nullptr, "null output pointer");
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

// .fmi bucket records (n_buckets x 64 B, host) -> device lines of ix's layout.
static uint8_t* upload_lines(fmg_index* ix, const void* bucket_records) {
  uint8_t* lines = nullptr;
  uint32_t bad = 0;
  const uint64_t n_buckets = ix->n_buckets;
  with_words(ix, [&](auto wt) {
    constexpr int W = decltype(wt)::value;
    ix->n_lines = (n_buckets * 128 + fmg::LineTraits<W>::kChars - 1) / fmg::LineTraits<W>::kChars;
    FMG_CK(dmalloc(&lines, ix->n_lines * fmg::LineTraits<W>::kBytes));
    uint64_t* staging = nullptr;
    uint32_t* err = nullptr;
    FMG_CK(cudaMalloc(&staging, n_buckets * 64 + 64));
    err = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(staging) + n_buckets * 64);
    FMG_CK(cudaMemcpy(staging, bucket_records, n_buckets * 64, cudaMemcpyHostToDevice));
    FMG_CK(cudaMemset(err, 0, sizeof(uint32_t)));
    fmg::k_build_lines<W><<<unsigned((ix->n_lines + 255) / 256), 256>>>(staging, n_buckets, lines, ix->n_lines,
                                                                         err);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&bad, err, sizeof(bad), cudaMemcpyDeviceToHost);
    cudaFree(staging);
    if (e != cudaSuccess) dfree(lines);
    FMG_CK(e);
  });
  if (bad != 0) dfree(lines);
  FMG_REQUIRE(bad == 0, "bucket base does not fit 32 bits");
  return lines;
}

int fmg_index_create(int device, const void* bucket_records, uint64_t n_buckets, uint64_t n, uint64_t sentinel_row,
                     const uint64_t c[5], fmg_index** out) {
  return fmg::guard([&] {
    FMG_REQUIRE(out != nullptr && bucket_records != nullptr && c != nullptr, "null argument");
    *out = nullptr;
    FMG_REQUIRE(n >= 1, "index covers an empty reference");
    FMG_REQUIRE(n + 1 < 0xFFFFFFFFull, "reference too long for 32-bit rows");
    FMG_REQUIRE(n_buckets == (n + 1 + 127) / 128, "bucket count does not match n");
    FMG_REQUIRE(sentinel_row <= n, "sentinel row outside [0, n]");
    FMG_REQUIRE(c[0] == 0 && c[4] == n, "C table endpoints wrong");
    for (int s = 0; s < 4; ++s) FMG_REQUIRE(c[s] <= c[s + 1], "C table not non-decreasing");
    int ndev = 0;
    FMG_CK(cudaGetDeviceCount(&ndev));
    FMG_REQUIRE(device >= 0 && device < ndev, "CUDA device ordinal out of range");
    DeviceScope scope(device);
    auto* ix = new fmg_index();
    try {
      ix->device = device;
      ix->n = n;
      ix->sentinel_row = sentinel_row;
      for (int s = 0; s < 5; ++s) ix->c[s] = c[s];
      ix->n_buckets = n_buckets;
      ix->words = choose_words(n_buckets);
      ix->sms = fmg::sm_count(device);
      ix->lines = upload_lines(ix, bucket_records);
      if (ix->n_lines * 32 > chunk_min_line_bytes() && ix->n_lines * 32 <= chunk_max_line_bytes()) {
        ix->chunk_sectors = chunk_sectors_default();
        ix->chunks = build_chunks(ix, bucket_records, ix->n_chunks);
      }
      // Allow the stream-ordered pool to keep freed blocks (host entry points
      // allocate per call).
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      *out = ix;
    } catch (...) {
      fmg_index_destroy(ix);
      throw;
    }
  });
}

int fmg_index_set_reverse(fmg_index* ix, const void* bucket_records, uint64_t n_buckets, uint64_t sentinel_row) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(bucket_records != nullptr, "null argument");
    FMG_REQUIRE(n_buckets == ix->n_buckets, "reverse index bucket count does not match the index");
    FMG_REQUIRE(sentinel_row <= ix->n, "sentinel row outside [0, n]");
    fmg::DeviceScope scope(ix->device);
    std::lock_guard<std::mutex> lock(ix->attach_mu);
    if (ix->rev_lines.load(std::memory_order_acquire)) return;  // attached once; the index is immutable
    uint8_t* rev = upload_lines(ix, bucket_records);
    ix->rev_sentinel_row = sentinel_row;
    DevBuf<uint32_t> tail(16, nullptr);
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      fmg::k_tail_keys<W><<<1, 32>>>(ix->view(), 16u, tail.ptr);
    });
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(ix->tail, tail.ptr, sizeof(ix->tail), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) dfree(rev);
    FMG_CK(e);
    ix->rev_lines.store(rev, std::memory_order_release);  // publishes rev_sentinel_row and tail too
  });
}

int fmg_index_has_reverse(const fmg_index* ix, int* has) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(has != nullptr, "null argument");
    *has = ix->rev_lines.load(std::memory_order_acquire) != nullptr;
  });
}

int fmg_index_set_samples(fmg_index* ix, const uint64_t* sa_samples, uint64_t count) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(sa_samples != nullptr, "null argument");
    FMG_REQUIRE(count == ix->n / 32 + 1, "sample count does not match n");
    std::vector<uint32_t> s32(count);
    for (uint64_t i = 0; i < count; ++i) {
      FMG_REQUIRE(sa_samples[i] <= ix->n, "suffix-array sample out of range");
      s32[i] = uint32_t(sa_samples[i]);
    }
    fmg::DeviceScope scope(ix->device);
    std::lock_guard<std::mutex> lock(ix->attach_mu);
    if (ix->samples.load(std::memory_order_acquire)) return;  // attached once; the index is immutable
    uint32_t* d = nullptr;
    FMG_CK(dmalloc(&d, count * sizeof(uint32_t)));
    const cudaError_t e = cudaMemcpy(d, s32.data(), count * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) dfree(d);
    FMG_CK(e);
    ix->n_samples = count;
    ix->samples.store(d, std::memory_order_release);
  });
}

int fmg_index_info(const fmg_index* ix, uint64_t* n, int* device, uint64_t* device_bytes) {
  return fmg::guard([&] {
    check_index(ix);
    if (n) *n = ix->n;
    if (device) *device = ix->device;
    if (device_bytes) {
      uint64_t lb = 0;
      with_words(ix, [&](auto wt) { lb = fmg::LineTraits<decltype(wt)::value>::kBytes; });
      const bool rev = ix->rev_lines.load(std::memory_order_acquire) != nullptr;
      const bool smp = ix->samples.load(std::memory_order_acquire) != nullptr;
      *device_bytes = ix->n_lines * lb * (rev ? 2 : 1) + (smp ? ix->n_samples * 4 : 0) +
                      ix->n_chunks * 32ull * uint64_t(ix->chunk_sectors);
    }
  });
}

void fmg_index_destroy(fmg_index* ix) {
  if (!ix) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ix->device);
  dfree(ix->lines);
  dfree(ix->chunks);
  dfree(ix->lut);
  dfree(ix->lut_r);
  dfree(ix->lut_x);
  dfree(ix->flt_bits);
  dfree(ix->ep_table);
  dfree(ix->rev_lines.load());
  dfree(ix->samples.load());
  if (prev >= 0) cudaSetDevice(prev);
  delete ix;
}

int fmg_occ_pair(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, uint32_t* status,
                 void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    launch_occ_pair(ix, kl, count, out, as_stream(stream), status);
  });
}

// Tuning hook (not part of include/fmgpu.h): same as fmg_occ_pair with an
// explicit pairs-per-thread and block size.
int fmgx_occ_pair_tuned(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out, void* stream,
                        int per, int threads) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    launch_occ_pair(ix, kl, count, out, as_stream(stream), nullptr, per, threads);
  });
}

// Work-counting variant of fmg_exact_packed (not part of include/fmgpu.h;
// bench.py's algorithmic-bytes figure): synchronous, returns the Occ steps
// executed and the 32-byte lines they fetched.
int fmgx_exact_packed_work(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count,
                           uint32_t* kl_out, void* stream, uint64_t* steps, uint64_t* lines) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(m >= 1 && m <= 32, "packed patterns need 1 <= m <= 32");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = as_stream(stream);
    DevBuf<unsigned long long> ctr(2, s);
    FMG_CK(cudaMemsetAsync(ctr.ptr, 0, 2 * sizeof(unsigned long long), s));
    launch_exact_packed(ix, packed, m, count, kl_out, s, ctr.ptr);
    unsigned long long h[2];
    FMG_CK(cudaMemcpyAsync(h, ctr.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    FMG_CK(cudaStreamSynchronize(s));
    if (steps) *steps = h[0];
    if (lines) *lines = h[1];
  });
}

// Layout the Occ-step kernel reads (not part of include/fmgpu.h; bench.py's
// algorithmic-bytes figure): 0 = 32-byte lines, else the sectors per chunk
// of the chunk layout (2: 64-byte, 4: 128-byte chunks).
int fmgx_occ_layout(const fmg_index* ix, int* chunked) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(chunked != nullptr, "null argument");
    *chunked = (ix->chunks != nullptr && !chunk_off()) ? ix->chunk_sectors : 0;
  });
}

// Lines fetched by a bounded-difference search (companion of fmg_matches_steps).
int fmgx_matches_lines(const fmg_matches* m, uint64_t* lines) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr && lines != nullptr, "null argument");
    *lines = m->lines;
  });
}

// Kernels of this library a bounded-difference search launched (counted by
// the flat engine's path; 0 when the engine does not count).
int fmgx_matches_launches(const fmg_matches* m, uint64_t* launches) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr && launches != nullptr, "null argument");
    *launches = m->launches;
  });
}

// Builds the prefix / k-mer table now instead of on the first large call
// (bench.py reports its build time and size apart from the timed region).
int fmgx_prefix_table(const fmg_index* ix, uint32_t* k_out, uint64_t* bytes_out) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    const PrefixTable pt = prefix_table(ix, 1u << 20, nullptr);
    if (k_out) *k_out = pt.k;
    if (bytes_out) *bytes_out = pt.base ? PrefixTable::off64(pt.k + 1) * sizeof(uint2) : 0;
  });
}

// Builds the exact search's k-mer table now (kmer_table: the prefix table's
// level K, or the level-(K + 1) extension); reports its K and the bytes of
// the extension (0 when exact search uses level K of the prefix table).
int fmgx_kmer_table(const fmg_index* ix, uint32_t* k_out, uint64_t* ext_bytes_out) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    const KmerTable kt = kmer_table(ix, 1u << 20, nullptr);
    if (k_out) *k_out = kt.k;
    if (ext_bytes_out) *ext_bytes_out = ix->lut_x ? (uint64_t(1) << (2 * ix->lut_x_k)) * sizeof(uint2) : 0;
  });
}

// Reporting hook: the flat engine's presence filter as built so far (all zero
// when none): window length B, group width G, copies, bytes.
int fmgx_flat_filter_info(const fmg_index* ix, uint32_t* b_out, uint32_t* g_out, uint32_t* copies_out,
                          uint64_t* bytes_out) {
  return fmg::guard([&] {
    check_index(ix);
    std::lock_guard<std::mutex> lock(const_cast<fmg_index*>(ix)->lut_mu);
    const bool have = ix->flt_bits != nullptr;
    if (b_out) *b_out = have ? ix->flt_B : 0;
    if (g_out) *g_out = have ? ix->flt_G : 0;
    if (copies_out) *copies_out = have ? ix->flt_NO : 0;
    if (bytes_out) *bytes_out = have ? (uint64_t(1) << (2 * ix->flt_B)) / 8 * ix->flt_NO : 0;
  });
}

// Tuning hook: L2 fetch granularity of the current context on `device`
// (cudaLimitMaxL2FetchGranularity; 32 = fetch exactly the 32-byte sector a
// line load needs).  Returns the previous value in *prev.
int fmgx_set_l2_fetch_granularity(int device, int bytes, int* prev) {
  return fmg::guard([&] {
    fmg::DeviceScope scope(device);
    size_t old = 0;
    FMG_CK(cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity));
    if (prev) *prev = int(old);
    if (bytes >= 0) FMG_CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(bytes)));
  });
}

// Measured random 32-byte fetches per second on `device` over `bytes` of
// memory (>> L2), best of 3 launches of `count` reads.  Used by bench.py as
// the request roofline of HBM-resident Occ steps.
int fmgx_random_fetch_rate(int device, uint64_t bytes, uint64_t count, double* rate) {
  return fmg::guard([&] {
    FMG_REQUIRE(rate != nullptr && bytes >= 32 && count > 0, "bad argument");
    fmg::DeviceScope scope(device);
    uint8_t* buf = nullptr;
    unsigned long long* sink = nullptr;
    FMG_CK(cudaMalloc(&buf, bytes));
    FMG_CK(cudaMalloc(&sink, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    cudaError_t err = cudaMemset(buf, 1, bytes);
    for (int r = 0; r < 4 && err == cudaSuccess; ++r) {
      cudaEventRecord(e0);
      fmg::k_random_fetch<<<unsigned((count + 255) / 256), 256>>>(buf, bytes / 32, count, uint64_t(r) * 7919, sink);
      cudaEventRecord(e1);
      err = cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0) best = std::min(best, ms);  // first launch is warm-up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(sink);
    FMG_CK(err);
    *rate = double(count) / (double(best) * 1e-3);
  });
}

int fmg_occ_pair_host(const fmg_index* ix, const uint32_t* kl, uint64_t count, uint32_t* out) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    if (count == 0) return;
    // FMG_OCC_ZEROCOPY=1 (A/B): pinned buffers read and written by the kernel itself, no staging;
    // slower for a whole config-1 step (1.54 vs 1.68 G steps/s, profiles/r02_ab_zerocopy.log): off
    if (const char* e = std::getenv("FMG_OCC_ZEROCOPY")) {
      if (std::atoi(e) != 0 && pinned_host(kl) && pinned_host(out)) {
        cudaStream_t s0 = host_stream(ix->device, 0);
        CallStatus st(nullptr, s0);
        launch_occ_pair(ix, kl, count, out, s0, st.word);
        st.raise_if_set(s0, "Occ position out of range or pair out of order");
        return;
      }
    }
    uint64_t chunk_log2 = 20;  // 2^20 pairs per chunk: 1.676 G steps/s e2e on config 1 against 1.662 G at 2^21, 1.619 G at 2^22 (profiles/r02_ab_e2e_chunk.log)
    if (const char* e = std::getenv("FMG_OCC_HOST_CHUNK_LOG2")) chunk_log2 = uint64_t(std::min(26, std::max(12, std::atoi(e))));  // A/B
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << chunk_log2);
    cudaStream_t s0 = host_stream(ix->device, 0);
    CallStatus st(nullptr, s0);
    FMG_CK(cudaStreamSynchronize(s0));  // the word is zeroed before any slot's kernel reads it
    pipeline_host(ix->device, count, std::max<uint64_t>(chunk, 1), 8, 32, kl, out,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_occ_pair(ix, static_cast<const uint32_t*>(din), len, static_cast<uint32_t*>(dout), s,
                                    st.word);
                  });
    st.raise_if_set(s0, "Occ position out of range or pair out of order");
  });
}

int fmg_exact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count, uint32_t* kl_out,
              void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    fmg::DeviceScope scope(ix->device);
    launch_exact_codes(ix, codes, offsets, count, kl_out, as_stream(stream), nullptr);
  });
}

int fmg_exact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, uint32_t* kl_out,
                     void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    fmg::DeviceScope scope(ix->device);
    launch_exact_packed(ix, packed, m, count, kl_out, as_stream(stream), nullptr);
  });
}

int fmg_exact_host(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                   uint32_t* kl_out) {
  return fmg::guard([&] {
    check_index(ix);
    if (count == 0) return;
    FMG_REQUIRE(offsets[0] == 0 && offsets[count] >= count, "pattern offsets must start at 0; patterns non-empty");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = host_stream(ix->device, 0);
    try {
      DevBuf<uint8_t> dc(offsets[count], s);
      DevBuf<uint64_t> doff(count + 1, s);
      DevBuf<uint32_t> dout(2 * count, s);
      FMG_CK(cudaMemcpyAsync(dc.ptr, codes, offsets[count], cudaMemcpyHostToDevice, s));
      FMG_CK(cudaMemcpyAsync(doff.ptr, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, s));
      validate_patterns_device(dc.ptr, doff.ptr, count, s);
      launch_exact_codes(ix, dc.ptr, doff.ptr, count, dout.ptr, s, nullptr);
      FMG_CK(cudaMemcpyAsync(kl_out, dout.ptr, 2 * count * 4, cudaMemcpyDeviceToHost, s));
      FMG_CK(cudaStreamSynchronize(s));
    } catch (...) {
      cudaStreamSynchronize(s);
      throw;
    }
    FMG_CK(cudaStreamSynchronize(s));
  });
}

int fmg_exact_packed_host(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count,
                          uint32_t* kl_out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    // Small batches in pinned host buffers: the kernel reads the patterns and
    // writes the intervals through the host mappings themselves — one launch
    // and one synchronisation instead of two staging allocations, two copies
    // and their launches (config 0, 10,000 patterns: 45 -> ~20 us per call).
    // FMG_EXACT_ZEROCOPY=0 keeps the staged pipeline (A/B).
    static const bool zc_on = [] {
      const char* e = std::getenv("FMG_EXACT_ZEROCOPY");
      return e == nullptr || std::atoi(e) != 0;
    }();
    if (zc_on && count <= (1u << 16) && pinned_host(packed) && pinned_host(kl_out)) {
      cudaStream_t s = host_stream(ix->device, 0);
      launch_exact_packed(ix, packed, m, count, kl_out, s, nullptr);
      FMG_CK(cudaStreamSynchronize(s));
      return;
    }
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 22);
    pipeline_host(ix->device, count, chunk, 8, 8, packed, kl_out,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_exact_packed(ix, static_cast<const uint64_t*>(din), m, len, static_cast<uint32_t*>(dout),
                                        s, nullptr);
                  });
  });
}

int fmg_inexact_wants_reverse(const fmg_index* ix, uint64_t count, uint64_t max_len, int max_diff, int* wants) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(wants != nullptr, "null output pointer");
    *wants = 0;
    if (max_diff != 1 || count < 1024) return;  // only the bidirectional z = 1 engines read a reverse index
    fmg::DeviceScope scope(ix->device);
    const bool lut_off = [] {
      const char* e = std::getenv("FMG_INEXACT_LUT");
      return e != nullptr && std::atoi(e) == 0;
    }();
    const PrefixTable pt = lut_off ? PrefixTable{} : prefix_table(ix, count, nullptr);
    *wants = flat_choice(ix, count, max_len, 1u, pt, nullptr).use ? 0 : 1;
  });
}

int fmg_inexact(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count, int max_diff,
                fmg_matches** out, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = as_stream(stream);
    static const bool trace = std::getenv("FMG_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t max_len = validate_patterns_device(codes, offsets, count, s);
    const auto t1 = std::chrono::steady_clock::now();
    *out = run_inexact(ix, codes, offsets, count, max_len, max_diff, s);
    if (trace) {
      const auto t2 = std::chrono::steady_clock::now();
      fprintf(stderr, "[fmg] fmg_inexact host time: validate %.3f ms, search %.3f ms\n",
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  });
}

int fmg_inexact_host(const fmg_index* ix, const uint8_t* codes, const uint64_t* offsets, uint64_t count,
                     int max_diff, fmg_matches** out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
    if (count > 0)
      FMG_REQUIRE(offsets[0] == 0 && offsets[count] >= count, "pattern offsets must start at 0; patterns non-empty");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = host_stream(ix->device, 0);
    try {
      DevBuf<uint8_t> dc(count ? offsets[count] : 0, s);
      DevBuf<uint64_t> doff(count + 1, s);
      if (count) {
        FMG_CK(cudaMemcpyAsync(dc.ptr, codes, offsets[count], cudaMemcpyHostToDevice, s));
        FMG_CK(cudaMemcpyAsync(doff.ptr, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, s));
      }
      const uint64_t max_len = validate_patterns_device(dc.ptr, doff.ptr, count, s);
      *out = run_inexact(ix, dc.ptr, doff.ptr, count, max_len, max_diff, s);
    } catch (...) {
      cudaStreamSynchronize(s);
      throw;
    }
    FMG_CK(cudaStreamSynchronize(s));
  });
}

int fmg_inexact_packed(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, int max_diff,
                       fmg_matches** out, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    fmg::DeviceScope scope(ix->device);
    *out = run_inexact(ix, nullptr, nullptr, count, m, max_diff, as_stream(stream), packed);
  });
}

int fmg_inexact_packed_host(const fmg_index* ix, const uint64_t* packed, uint32_t m, uint64_t count, int max_diff,
                            fmg_matches** out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(out != nullptr, "null output pointer");
    *out = nullptr;
    FMG_REQUIRE(m >= 1 && m <= 32, "packed pattern length must be in [1, 32]");
    FMG_REQUIRE(max_diff >= 0, "difference budget is negative");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = host_stream(ix->device, 0);
    try {
      DevBuf<uint64_t> dp(count, s);
      if (count) FMG_CK(cudaMemcpyAsync(dp.ptr, packed, count * 8, cudaMemcpyHostToDevice, s));
      *out = run_inexact(ix, nullptr, nullptr, count, m, max_diff, s, dp.ptr);
    } catch (...) {
      cudaStreamSynchronize(s);
      throw;
    }
    FMG_CK(cudaStreamSynchronize(s));
  });
}

int fmg_matches_size(const fmg_matches* m, uint64_t* total, uint64_t* patterns) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr, "null matches handle");
    if (total) *total = m->total;
    if (patterns) *patterns = m->patterns;
  });
}

int fmg_matches_steps(const fmg_matches* m, uint64_t* steps) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr && steps != nullptr, "null argument");
    *steps = m->steps;
  });
}

int fmg_matches_copy(const fmg_matches* m, uint64_t* row_offsets, uint32_t* k, uint32_t* l, uint8_t* diffs,
                     int to_host) {
  return fmg::guard([&] {
    FMG_REQUIRE(m != nullptr, "null matches handle");
    fmg::DeviceScope scope(m->device);
    const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    // the calling thread's own copy stream, never the legacy stream: a result
    // set copied out by one thread while another searches must not queue
    // behind, or in front of, that search
    cudaStream_t s = host_stream(m->device, 1);
    if (row_offsets) FMG_CK(cudaMemcpyAsync(row_offsets, m->row_off, (m->patterns + 1) * 8, kind, s));
    if (m->total && m->kl && (k || l)) {  // packed k | l: split on the device, then copy
      DevBuf<uint32_t> dk(to_host && k ? m->total : 0, s), dl(to_host && l ? m->total : 0, s);
      uint32_t* ok = to_host ? dk.ptr : k;
      uint32_t* ol = to_host ? dl.ptr : l;
      fmg::k_split_kl<<<unsigned(std::min<uint64_t>((m->total + 255) / 256, 148 * 16)), 256, 0, s>>>(
          m->kl, m->total, k ? ok : nullptr, l ? ol : nullptr);
      FMG_CK(cudaGetLastError());
      if (to_host && k) FMG_CK(cudaMemcpyAsync(k, dk.ptr, m->total * 4, cudaMemcpyDeviceToHost, s));
      if (to_host && l) FMG_CK(cudaMemcpyAsync(l, dl.ptr, m->total * 4, cudaMemcpyDeviceToHost, s));
      if (m->total && diffs) FMG_CK(cudaMemcpyAsync(diffs, m->diffs, m->total, kind, s));
      FMG_CK(cudaStreamSynchronize(s));  // before dk / dl go out of scope
      return;
    } else if (m->total) {
      if (k) FMG_CK(cudaMemcpyAsync(k, m->k, m->total * 4, kind, s));
      if (l) FMG_CK(cudaMemcpyAsync(l, m->l, m->total * 4, kind, s));
    }
    if (m->total && diffs) FMG_CK(cudaMemcpyAsync(diffs, m->diffs, m->total, kind, s));
    FMG_CK(cudaStreamSynchronize(s));
  });
}

void fmg_matches_free(fmg_matches* m) {
  if (!m) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  // pool allocations (run_inexact synchronised its stream before returning)
  // stream-ordered frees on the stream the search allocated on: the pool
  // reuses the blocks for that stream's next call without any cross-stream
  // dependency (freeing on the legacy stream made the next call map memory)
  afree(m->row_off, m->stream);
  afree(m->k, m->stream);
  afree(m->l, m->stream);
  afree(m->kl, m->stream);
  afree(m->diffs, m->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

int fmg_psi_inverse(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint8_t* out_sym, uint32_t* out_row,
                    uint32_t* status, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    with_words(ix, [&](auto wt) {
      fmg::k_psi<decltype(wt)::value><<<unsigned((count + 255) / 256), 256, 0, as_stream(stream)>>>(
          ix->view(), rows, count, out_sym, out_row, status);
    });
    FMG_CK(cudaGetLastError());
  });
}

int fmg_locate_rows(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos, uint32_t* status,
                    void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(ix->samples.load(std::memory_order_acquire) != nullptr,
                "index has no suffix-array samples (fmg_index_set_samples)");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    launch_locate(ix, rows, count, out_pos, as_stream(stream), status);
    FMG_CK(cudaGetLastError());
  });
}

int fmg_locate_rows_host(const fmg_index* ix, const uint32_t* rows, uint64_t count, uint32_t* out_pos) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(ix->samples.load(std::memory_order_acquire) != nullptr,
                "index has no suffix-array samples (fmg_index_set_samples)");
    if (count == 0) return;
    fmg::DeviceScope scope(ix->device);
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 22);
    cudaStream_t s0 = host_stream(ix->device, 0);
    CallStatus st(nullptr, s0);
    FMG_CK(cudaStreamSynchronize(s0));
    pipeline_host(ix->device, count, chunk, 4, 4, rows, out_pos,
                  [&](void* din, uint64_t len, void* dout, cudaStream_t s) {
                    launch_locate(ix, static_cast<const uint32_t*>(din), len, static_cast<uint32_t*>(dout), s,
                                  st.word);
                    FMG_CK(cudaGetLastError());
                  });
    st.raise_if_set(s0, "row out of range");
  });
}

int fmg_reconstruct_text(const fmg_index* ix, uint8_t* codes_out, uint32_t* status, void* stream) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(codes_out != nullptr, "null output pointer");
    FMG_REQUIRE(ix->samples.load(std::memory_order_acquire) != nullptr,
                "index has no suffix-array samples (fmg_index_set_samples)");
    fmg::DeviceScope scope(ix->device);
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      const uint64_t ns = ix->n / 32 + 1;
      const unsigned blocks = wave_blocks(ix, (const void*)fmg::k_reconstruct<W>, 256, ns);
      fmg::k_reconstruct<W><<<blocks, 256, 0, as_stream(stream)>>>(ix->view(), ns, codes_out, status);
    });
    FMG_CK(cudaGetLastError());
  });
}

int fmg_reconstruct_text_host(const fmg_index* ix, uint8_t* codes_out) {
  return fmg::guard([&] {
    check_index(ix);
    FMG_REQUIRE(codes_out != nullptr, "null output pointer");
    FMG_REQUIRE(ix->samples.load(std::memory_order_acquire) != nullptr,
                "index has no suffix-array samples (fmg_index_set_samples)");
    fmg::DeviceScope scope(ix->device);
    cudaStream_t s = host_stream(ix->device, 0);
    CallStatus st(nullptr, s);
    DevBuf<uint8_t> text(ix->n, s);
    with_words(ix, [&](auto wt) {
      constexpr int W = decltype(wt)::value;
      const uint64_t ns = ix->n / 32 + 1;
      const unsigned blocks = wave_blocks(ix, (const void*)fmg::k_reconstruct<W>, 256, ns);
      fmg::k_reconstruct<W><<<blocks, 256, 0, s>>>(ix->view(), ns, text.ptr, st.word);
    });
    FMG_CK(cudaGetLastError());
    FMG_CK(cudaMemcpyAsync(codes_out, text.ptr, ix->n, cudaMemcpyDeviceToHost, s));
    st.raise_if_set(s, "text reconstruction failed");
  });
}

// ---- bucket-level rank kernels (kernels.py:125-292) ----

static unsigned grid_for(uint64_t count, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (count + threads - 1) / threads;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(sms) * 16)));
}

static void launch_bucket_count(const uint8_t* blocks, const uint32_t* prefix_lens, const uint8_t* symbols,
                                uint64_t count, int method, uint32_t* out, uint32_t* status, cudaStream_t s) {
  FMG_REQUIRE(method == 0 || method == 1, "bucket method must be 0 (popcount) or 1 (nibble)");
  FMG_REQUIRE(reinterpret_cast<uintptr_t>(blocks) % 32 == 0, "bucket blocks must be 32-byte aligned");
  if (method == 0)
    fmg::k_bucket_count<0><<<grid_for(count, 256), 256, 0, s>>>(blocks, prefix_lens, symbols, count, out, status);
  else
    fmg::k_bucket_count<1><<<grid_for(count, 256), 256, 0, s>>>(blocks, prefix_lens, symbols, count, out, status);
  FMG_CK(cudaGetLastError());
}

int fmg_bucket_count(const uint8_t* blocks, const uint32_t* prefix_lens, const uint8_t* symbols, uint64_t count,
                     int method, uint32_t* out, uint32_t* status, void* stream) {
  return fmg::guard([&] {
    if (count == 0) return;
    FMG_REQUIRE(blocks && prefix_lens && out, "null argument");
    launch_bucket_count(blocks, prefix_lens, symbols, count, method, out, status, as_stream(stream));
  });
}

int fmg_bucket_count_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens, const uint8_t* symbols,
                          uint64_t count, int method, uint32_t* out) {
  return fmg::guard([&] {
    if (count == 0) return;
    FMG_REQUIRE(blocks && prefix_lens && out, "null argument");
    fmg::DeviceScope scope(device);
    cudaStream_t s = host_stream(device, 0);
    CallStatus st(nullptr, s);
    DevBuf<uint8_t> d_blocks(count * 32, s), d_sym(symbols ? count : 0, s);
    DevBuf<uint32_t> d_pl(count, s), d_out(count * (symbols ? 1 : 4), s);
    FMG_CK(cudaMemcpyAsync(d_blocks.ptr, blocks, count * 32, cudaMemcpyHostToDevice, s));
    FMG_CK(cudaMemcpyAsync(d_pl.ptr, prefix_lens, count * 4, cudaMemcpyHostToDevice, s));
    if (symbols) FMG_CK(cudaMemcpyAsync(d_sym.ptr, symbols, count, cudaMemcpyHostToDevice, s));
    launch_bucket_count(d_blocks.ptr, d_pl.ptr, symbols ? d_sym.ptr : nullptr, count, method, d_out.ptr, st.word, s);
    FMG_CK(cudaMemcpyAsync(out, d_out.ptr, count * 4 * (symbols ? 1 : 4), cudaMemcpyDeviceToHost, s));
    st.raise_if_set(s, "prefix_len outside [0, 128] or symbol code outside [0, 4)");
  });
}

int fmg_bucket_mask_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens, uint64_t count,
                         uint8_t* out) {
  return fmg::guard([&] {
    if (count == 0) return;
    FMG_REQUIRE(blocks && prefix_lens && out, "null argument");
    fmg::DeviceScope scope(device);
    cudaStream_t s = host_stream(device, 0);
    CallStatus st(nullptr, s);
    DevBuf<uint8_t> d_blocks(count * 32, s), d_out(count * 32, s);
    DevBuf<uint32_t> d_pl(count, s);
    FMG_CK(cudaMemcpyAsync(d_blocks.ptr, blocks, count * 32, cudaMemcpyHostToDevice, s));
    FMG_CK(cudaMemcpyAsync(d_pl.ptr, prefix_lens, count * 4, cudaMemcpyHostToDevice, s));
    fmg::k_bucket_mask<<<grid_for(count, 256), 256, 0, s>>>(d_blocks.ptr, d_pl.ptr, count, d_out.ptr, st.word);
    FMG_CK(cudaGetLastError());
    FMG_CK(cudaMemcpyAsync(out, d_out.ptr, count * 32, cudaMemcpyDeviceToHost, s));
    st.raise_if_set(s, "prefix_len outside [0, 128]");
  });
}

int fmg_bucket_nibble_trace_host(int device, const uint8_t* blocks, const uint32_t* prefix_lens,
                                 const uint8_t* symbols, uint64_t count, uint64_t* trace) {
  return fmg::guard([&] {
    if (count == 0) return;
    FMG_REQUIRE(blocks && prefix_lens && symbols && trace, "null argument");
    fmg::DeviceScope scope(device);
    cudaStream_t s = host_stream(device, 0);
    CallStatus st(nullptr, s);
    DevBuf<uint8_t> d_blocks(count * 32, s), d_sym(count, s);
    DevBuf<uint32_t> d_pl(count, s);
    DevBuf<uint64_t> d_tr(count * 15, s);
    FMG_CK(cudaMemcpyAsync(d_blocks.ptr, blocks, count * 32, cudaMemcpyHostToDevice, s));
    FMG_CK(cudaMemcpyAsync(d_pl.ptr, prefix_lens, count * 4, cudaMemcpyHostToDevice, s));
    FMG_CK(cudaMemcpyAsync(d_sym.ptr, symbols, count, cudaMemcpyHostToDevice, s));
    fmg::k_bucket_nibble_trace<<<unsigned((count + 127) / 128), 128, 0, s>>>(d_blocks.ptr, d_pl.ptr, d_sym.ptr,
                                                                             count, d_tr.ptr, st.word);
    FMG_CK(cudaGetLastError());
    FMG_CK(cudaMemcpyAsync(trace, d_tr.ptr, count * 15 * 8, cudaMemcpyDeviceToHost, s));
    st.raise_if_set(s, "prefix_len outside [0, 128] or symbol code outside [0, 4)");
  });
}

// Guard-mode self test (not part of include/fmgpu.h): reads the first u32
// past the (32-byte-rounded) end of a guarded 1000-byte buffer.  Under FMG_GUARD=1 the read must
// fault; *faulted = 1 when the launch reported an error.  The fault poisons
// the CUDA context, so callers run this in a throwaway process.
__global__ void k_guard_probe(const uint32_t* p, uint32_t idx, uint32_t* sink) { *sink = p[idx]; }

int fmgx_guard_selftest(int device, int* faulted) {
  return fmg::guard([&] {
    FMG_REQUIRE(faulted != nullptr, "null argument");
    fmg::DeviceScope scope(device);
    uint32_t* buf = nullptr;
    uint32_t* sink = nullptr;
    FMG_CK(dmalloc(&buf, 1000));
    FMG_CK(cudaMalloc(&sink, 4));
    FMG_CK(cudaMemset(buf, 0, 1000));
    k_guard_probe<<<1, 1>>>(buf, 256, sink);  // bytes 1024..1027: the first word past the rounded end
    cudaError_t e = cudaDeviceSynchronize();
    *faulted = e != cudaSuccess;
  });
}

int fmg_stream_sync(void* stream) {
  return fmg::guard([&] { FMG_CK(cudaStreamSynchronize(as_stream(stream))); });
}

}  // extern "C"
