// forge/cuda/copy.cuh — vcopy, the bandwidth-calibration kernel, and strided moves.
//
// Reference: prim::vcopy (primitives.hpp:305-341): grid-stride nitem-wide
// vload/vstore, scalar tail by the last thread (paper Fig. 1 / Listing 2).
// sm_100a: a grid of #SM x 4 CTAs, UNROLL independent 256-bit loads in flight
// per thread (ld.global.nc.L1::no_allocate.v8) then 256-bit stores; head and
// tail elements that do not fill a 32-byte vector are copied by the first
// threads.  When src and dst are not congruent modulo 32 bytes the copy falls
// back to element moves (still coalesced).
#pragma once

#include "forge/cuda/reduce.cuh"
#include "forge/cuda/tma.cuh"

namespace forge::cuda {

constexpr int kCopyThreads = 256;

template <class T, int UNROLL>
__global__ void __launch_bounds__(kCopyThreads)
    vcopy_kernel(const T* __restrict__ src, T* __restrict__ dst, uint64_t n, bool vec) {
  constexpr int VE = mr_vec_elems<T>();
  constexpr int VB = VE * int(sizeof(T));
  const uint64_t gtid = uint64_t(blockIdx.x) * kCopyThreads + threadIdx.x;
  const uint64_t gsize = uint64_t(gridDim.x) * kCopyThreads;
  if (!vec || VE == 1) {
    for (uint64_t i = gtid; i < n; i += gsize) dst[i] = src[i];
    return;
  }
  const uintptr_t addr = reinterpret_cast<uintptr_t>(src);
  uint64_t head = ((VB - (addr % VB)) % VB) / sizeof(T);
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / VE;
  const T* s = src + head;
  T* d = dst + head;
  constexpr uint64_t kChunk = uint64_t(kCopyThreads) * UNROLL;
  const uint64_t full = nvec / kChunk;
  for (uint64_t c = blockIdx.x; c < full; c += gridDim.x) {
    T x[UNROLL][VE];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      load_items<T, VE>(s + (c * kChunk + u * kCopyThreads + threadIdx.x) * VE, x[u]);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      store_items<T, VE>(d + (c * kChunk + u * kCopyThreads + threadIdx.x) * VE, x[u]);
  }
  for (uint64_t v = full * kChunk + gtid; v < nvec; v += gsize) {
    T x[VE];
    load_items<T, VE>(s + v * VE, x);
    store_items<T, VE>(d + v * VE, x);
  }
  const uint64_t tail0 = head + nvec * VE;
  const uint64_t extra = head + (n - tail0);
  for (uint64_t e = gtid; e < extra; e += gsize) {
    const uint64_t i = e < head ? e : tail0 + (e - head);
    dst[i] = src[i];
  }
}

// ---------------------------------------------------------------------------
// TMA bulk copy (the B200 path of vcopy for 16-byte-congruent buffers): one
// CTA per SM, one elected thread streams 32 KB chunks global -> shared ->
// global with cp.async.bulk through a ring of kBulkStages stages, keeping
// kBulkStages-1 loads in flight (~160 KB per SM, the Little's-law depth for
// read+write at HBM latency) while the stores drain behind them.  No register
// staging and no per-element instructions: the copy engine moves the bytes.

constexpr uint32_t kBulkChunk = 32u << 10;
constexpr int kBulkStages = 6;
constexpr int kBulkMaxStages = 12;
constexpr uint32_t kBulkDyn = kBulkStages * kBulkChunk;

__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* ssrc, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_load_1d(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Copies `bytes` (multiple of 16) from src to dst (both 16-byte aligned).
__global__ void __launch_bounds__(32, 1)
    bulk_copy_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, uint64_t bytes,
                     uint32_t chunk, int stages, bool hint) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  __shared__ __align__(8) uint64_t full[kBulkMaxStages];
  if (threadIdx.x != 0) return;
  const uint64_t nchunks = ceil_div(bytes, chunk);
  const uint64_t G = gridDim.x;
  const uint64_t mine = blockIdx.x < nchunks ? (nchunks - 1 - blockIdx.x) / G + 1 : 0;
  if (mine == 0) return;
  const uint64_t pol = hint ? policy_evict_first() : 0;
  for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  auto chunk_bytes = [&](uint64_t k) {
    const uint64_t off = (blockIdx.x + k * G) * uint64_t(chunk);
    return uint32_t(bytes - off < chunk ? bytes - off : chunk);
  };
  auto issue_load = [&](uint64_t k) {
    const int s = int(k % uint64_t(stages));
    const uint64_t off = (blockIdx.x + k * G) * uint64_t(chunk);
    const uint32_t b = chunk_bytes(k);
    mbar_arrive_expect_tx(&full[s], b);
    if (hint)
      bulk_load_1d(bulk_smem + size_t(s) * chunk, src + off, b, &full[s], pol);
    else
      tma_load_1d(bulk_smem + size_t(s) * chunk, src + off, b, &full[s]);
  };
  for (uint64_t k = 0; k < mine && k < uint64_t(stages); ++k) issue_load(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const int s = int(k % uint64_t(stages));
    mbar_wait(&full[s], uint32_t(k / uint64_t(stages)) & 1u);
    const uint64_t off = (blockIdx.x + k * G) * uint64_t(chunk);
    if (hint)
      bulk_store_1d(dst + off, bulk_smem + size_t(s) * chunk, chunk_bytes(k), pol);
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                   "r"(smem_addr(bulk_smem + size_t(s) * chunk)), "r"(chunk_bytes(k))
                   : "memory");
    tma_store_commit();
    // refill the stage of chunk k-1 once its store has read shared memory
    if (k >= 1 && k - 1 + uint64_t(stages) < mine) {
      bulk_wait_read<1>();
      issue_load(k - 1 + uint64_t(stages));
    }
  }
  bulk_wait_read<0>();
}

template <class T>
__global__ void strided_copy_kernel(const T* src, uint64_t sstride, T* dst, uint64_t dstride,
                                    uint64_t n) {
  const uint64_t gsize = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += gsize)
    dst[i * dstride] = src[i * sstride];
}

template <class T>
inline uint32_t copy_grid(uint64_t n) {
  const uint64_t per = uint64_t(kCopyThreads) * mr_vec_elems<T>() * 4;
  const uint64_t want = ceil_div(n, per);
  // One 32 KB chunk per CTA (no grid-stride loop) unless FORGE_COPY_GRID_PER_SM
  // caps the grid: measured 6.85 TB/s against 5.96 TB/s for a persistent
  // 4-CTA/SM grid and 6.49 TB/s for the driver's cudaMemcpy (profiles/).
  static const uint64_t per_sm = std::getenv("FORGE_COPY_GRID_PER_SM")
                                     ? std::strtoull(std::getenv("FORGE_COPY_GRID_PER_SM"), nullptr, 10)
                                     : (uint64_t(1) << 24);
  const uint64_t cap0 = uint64_t(device_props().sm_count) * per_sm;
  const uint64_t cap = cap0 < 0x7fffffffull ? cap0 : 0x7fffffffull;
  return uint32_t(want < 1 ? 1 : (want > cap ? cap : want));
}

template <class T>
cudaError_t launch_vcopy(const T* src, T* dst, uint64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  constexpr int VB = mr_vec_elems<T>() * int(sizeof(T));
  const bool vec = (reinterpret_cast<uintptr_t>(src) % VB) == (reinterpret_cast<uintptr_t>(dst) % VB) &&
                   (reinterpret_cast<uintptr_t>(src) % sizeof(T)) == 0;
  const uint64_t bytes = n * sizeof(T);
  static const bool bulk = std::getenv("FORGE_COPY_BULK") != nullptr;  // TMA bulk path (measured slower)
  if (bulk && bytes >= (8u << 20) && is_aligned(src, 16) && is_aligned(dst, 16) && bytes % 16 == 0) {
    // experiment knobs: FORGE_COPY_CHUNK_KB, FORGE_COPY_STAGES, FORGE_COPY_CTAS (per SM), FORGE_COPY_HINT
    static const uint32_t chunk = uint32_t(std::strtoul(std::getenv("FORGE_COPY_CHUNK_KB") ? std::getenv("FORGE_COPY_CHUNK_KB") : "32", nullptr, 10)) << 10;
    static const int stages = int(std::strtol(std::getenv("FORGE_COPY_STAGES") ? std::getenv("FORGE_COPY_STAGES") : "6", nullptr, 10));
    static const uint32_t ctas = uint32_t(std::strtoul(std::getenv("FORGE_COPY_CTAS") ? std::getenv("FORGE_COPY_CTAS") : "1", nullptr, 10));
    static const bool hint = std::getenv("FORGE_COPY_HINT") ? std::getenv("FORGE_COPY_HINT")[0] == '1' : true;
    static thread_local int done_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint32_t dyn = chunk * uint32_t(stages);
    if (done_dev != dev) {
      cudaFuncSetAttribute(bulk_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
      done_dev = dev;
    }
    const uint64_t chunks = ceil_div(bytes, chunk);
    const uint64_t cap = uint64_t(device_props().sm_count) * ctas;
    bulk_copy_kernel<<<uint32_t(chunks < cap ? chunks : cap), 32, dyn, stream>>>(
        reinterpret_cast<const unsigned char*>(src), reinterpret_cast<unsigned char*>(dst), bytes, chunk, stages,
        hint);
    return cudaGetLastError();
  }
  vcopy_kernel<T, 4><<<copy_grid<T>(n), kCopyThreads, 0, stream>>>(src, dst, n, vec);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_strided_copy(const T* src, uint64_t sstride, T* dst, uint64_t dstride,
                                uint64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (sstride == 1 && dstride == 1) return launch_vcopy(src, dst, n, stream);
  uint64_t grid = ceil_div(n, 256);
  const uint64_t cap = uint64_t(device_props().sm_count) * 8;
  if (grid > cap) grid = cap;
  strided_copy_kernel<T><<<uint32_t(grid), 256, 0, stream>>>(src, sstride, dst, dstride, n);
  return cudaGetLastError();
}

}  // namespace forge::cuda
