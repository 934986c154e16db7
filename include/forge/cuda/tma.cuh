// forge/cuda/tma.cuh — Tensor Memory Accelerator helpers for sm_100a.
//
// Host: builds CUtensorMap descriptors with cuTensorMapEncodeTiled, fetched
// through cudaGetDriverEntryPoint (no libcuda link needed).  Device: 2-D
// cp.async.bulk.tensor loads completing on an mbarrier.
//
// The primitives view a contiguous input as a byte matrix of 128-byte rows and
// load boxes of `box_rows` rows with CU_TENSOR_MAP_SWIZZLE_128B: inside every
// 1024-byte block, the 16-byte chunk c of row r lands at chunk c ^ (r & 7).  A
// thread that owns one row then reads its chunks IN ORDER with each quarter-warp
// touching 8 distinct bank groups — conflict-free without padding.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "forge/cuda/device.cuh"

namespace forge::cuda {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// rows x 128-byte matrix at `base` (16-byte aligned), boxes of box_rows rows.
// Encoded maps are cached per thread (8 entries, round robin): a driver
// encode per call is host latency a small scan would otherwise pay each time.
inline bool make_rows128_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t box_rows) {
  struct Entry {
    const void* base;
    uint64_t rows;
    uint32_t box;
    CUtensorMap map;
  };
  static thread_local Entry cache[8] = {};
  static thread_local unsigned next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* key = static_cast<const char*>(base) + (uint64_t(dev) << 56);  // device-qualified
  for (const Entry& e : cache)
    if (e.base == key && e.rows == rows && e.box == box_rows && rows != 0) {
      *map = e.map;
      return true;
    }
  auto enc = tensor_map_encoder();
  if (!enc || rows == 0 || !is_aligned(base, 16)) return false;
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const bool ok = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  if (ok) cache[next++ % 8] = Entry{key, rows, box_rows, *map};
  return ok;
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_addr(smem_dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

// L2 cache policies for the TMA's .L2::cache_hint operand: evict_last keeps a
// tile that will be read again soon (the lagged scan's re-read), evict_first
// marks a tile that is done with.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const CUtensorMap* map, int x, int y,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_addr(smem_dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, int x, int y, const void* smem_src,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   map),
               "r"(x), "r"(y), "r"(smem_addr(smem_src)), "l"(policy)
               : "memory");
}

// shared -> global 2-D tensor store (bulk-group completion).  Generic-proxy
// writes to the source must be made visible first: fence_proxy_async_smem().
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* smem_src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
               "r"(y), "r"(smem_addr(smem_src))
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Waits until the committed stores have finished READING shared memory.
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// L2 prefetch of one 2-D box (no shared memory, no barrier), with an L2
// eviction-priority policy.
__device__ __forceinline__ void tma_prefetch_2d_hint(const CUtensorMap* map, int x, int y, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile.L2::cache_hint [%0, {%1, %2}], %3;" ::"l"(map),
               "r"(x), "r"(y), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void prefetch_tensor_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// Byte offset of 16-byte chunk c of row r in a SWIZZLE_128B tile (1024-B aligned base).
__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace forge::cuda
