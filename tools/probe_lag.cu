// probe_lag.cu — development probe (not product): does a tile re-read D tiles
// after its first read still hit L2 under full HBM streaming?  This is the
// memory skeleton of a "lagged" scan (phase A of ticket k reads tile k, phase B
// re-reads tile k-D and writes it): if the re-read hits L2, HBM traffic stays
// 2n and the time matches a copy.
//   nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -I include -o tools/probe_lag tools/probe_lag.cu
#include <cstdio>
#include <cstdlib>

#include "forge/cuda/tma.cuh"

using namespace forge::cuda;

__device__ __forceinline__ uint64_t policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_hint(const CUtensorMap* map, int x, int y, const void* src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   map),
               "r"(x), "r"(y), "r"(smem_addr(src)), "l"(pol)
               : "memory");
}

constexpr int kThreads = 256;
constexpr uint32_t kTileBytes = 32768;

__global__ void __launch_bounds__(kThreads, 6)
    lag_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, uint32_t ntiles,
               uint32_t D, float* agg, int mode, int hint) {
  extern __shared__ unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ float red[kThreads / 32];
  unsigned char* buf = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t k = blockIdx.x;
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (k < ntiles && mode != 2) {  // phase A: first read + fold
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, kTileBytes);
      if (hint) tma_load_hint(buf, &tin, 0, int(k) * kThreads, &bar, policy_last());
      else tma_load_2d(buf, &tin, 0, int(k) * kThreads, &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 v = lds128(buf + swz128(threadIdx.x, c));
      s += __uint_as_float(v.x) + __uint_as_float(v.y) + __uint_as_float(v.z) + __uint_as_float(v.w);
    }
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(~0u, s, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0;
      for (int w = 0; w < kThreads / 32; ++w) t += red[w];
      agg[k] = t;
    }
  }
  const uint32_t j = mode == 2 ? k : k - D;
  if (k >= D && j < ntiles && mode != 1) {  // phase B: re-read + write
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, kTileBytes);
      if (hint) tma_load_hint(buf, &tin, 0, int(j) * kThreads, &bar, policy_first());
      else tma_load_2d(buf, &tin, 0, int(j) * kThreads, &bar);
    }
    mbar_wait(&bar, phase);
    if (threadIdx.x == 0) {
      if (hint) tma_store_hint(&tout, 0, int(j) * kThreads, buf, policy_first());
      else tma_store_2d(&tout, 0, int(j) * kThreads, buf);
      tma_store_commit();
      tma_store_wait_read();
    }
  }
}

int main(int argc, char** argv) {
  const uint64_t n = 1ull << 28;  // f32
  const uint64_t bytes = n * 4;
  const uint32_t ntiles = uint32_t(bytes / kTileBytes);
  char *in, *out;
  float* agg;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&agg, ntiles * 4);
  cudaMemset(in, 1, bytes);
  CUtensorMap tin, tout;
  make_rows128_map(&tin, in, bytes / 128, kThreads);
  make_rows128_map(&tout, out, bytes / 128, kThreads);
  const uint32_t dyn = kTileBytes + 1024;
  cudaFuncSetAttribute(lag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  cudaFuncSetAttribute(lag_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  // mode 2: plain TMA copy (read + write once); mode 1: phase A only (read);
  // mode 0: A + lagged B (read, re-read, write)
  struct Cfg {
    int mode;
    uint32_t D;
    int hint;
  } cfgs[] = {{2, 0, 0}, {1, 0, 0}, {0, 0, 0}, {0, 64, 0}, {0, 256, 0}, {0, 512, 0}, {0, 1024, 0}, {0, 1536, 0},
              {0, 2048, 0}, {0, 4096, 0}, {2, 0, 1}, {0, 256, 1}, {0, 512, 1}, {0, 1024, 1}, {0, 1536, 1},
              {0, 2048, 1}, {0, 4096, 1}};
  int idx = 0;
  for (const Cfg& c : cfgs) {
    if (only >= 0 && idx++ != only) continue;
    const uint32_t grid = c.mode == 0 ? ntiles + c.D : ntiles;
    for (int w = 0; w < 3; ++w) lag_kernel<<<grid, kThreads, dyn>>>(tin, tout, ntiles, c.D, agg, c.mode, c.hint);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      lag_kernel<<<grid, kThreads, dyn>>>(tin, tout, ntiles, c.D, agg, c.mode, c.hint);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double alg = c.mode == 1 ? double(bytes) : 2.0 * double(bytes);
    printf("{\"mode\": %d, \"D\": %u, \"hint\": %d, \"ms\": %.4f, \"alg_gbs\": %.1f}\n", c.mode, c.D, c.hint, best, alg / best / 1e6);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
