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
  // One 32 KB chunk per CTA (no grid-stride loop): measured 6.85 TB/s against
  // 5.96 TB/s for a persistent 4-CTA/SM grid, 6.18 TB/s for a TMA bulk-copy
  // ring and 6.49 TB/s for the driver's cudaMemcpy (profiles/r01).
  static const uint64_t per_sm = dev_knob("FORGE_COPY_GRID_PER_SM", 1u << 24);
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
