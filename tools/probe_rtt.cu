// probe_rtt.cu — development probe (not product): L2-hit round-trip latency of
// a state poll (ld.relaxed.gpu of a hot line) under full HBM streaming, seen
// from (a) an SM running the streaming CTAs and (b) an SM running nothing else.
// Decides whether a look-back service on a quiet SM can resolve tile carries
// faster than the tiles' own warps.
//   nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -I include -o tools/probe_rtt tools/probe_rtt.cu
#include <cstdio>
#include <cstdlib>

#include "forge/cuda/tma.cuh"

using namespace forge::cuda;

constexpr int kThreads = 256;
constexpr uint32_t kTileBytes = 32768;

__device__ __forceinline__ uint64_t gclock() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// TMA copy, one 32 KB tile per CTA; thread 0 of every CTA times one 32-lane
// poll round (warp 0) issued while its own tile is in flight.
__global__ void __launch_bounds__(kThreads, 6)
    stream_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                  const uint64_t* hot, unsigned long long* acc) {
  extern __shared__ unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar;
  unsigned char* buf = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t k = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bar, kTileBytes);
    tma_load_2d(buf, &tin, 0, int(k) * kThreads, &bar);
  }
  if (threadIdx.x < 32) {
    const uint64_t t0 = gclock();
    uint64_t v = ld_relaxed_gpu(hot + (k * 32 + threadIdx.x) % 4096 * 32);
    v = __reduce_or_sync(~0u, uint32_t(v));
    const uint64_t t1 = gclock();
    if (threadIdx.x == 0 && v != 12345) {
      atomicAdd(acc + 0, (unsigned long long)(t1 - t0));
      atomicAdd(acc + 1, 1ull);
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) {
    tma_store_2d(&tout, 0, int(k) * kThreads, buf);
    tma_store_commit();
    tma_store_wait_read();
  }
}

// One warp on its own SM (the CTA asks for all the shared memory, so nothing
// else co-resides): rounds of 32 independent polls, `batches` rounds in
// flight, for `dur_ns`.
__global__ void quiet_kernel(const uint64_t* hot, unsigned long long* acc, uint64_t dur_ns, int batches) {
  extern __shared__ unsigned char dyn[];
  if (threadIdx.x >= 32) return;
  const uint64_t start = gclock();
  uint64_t rounds = 0, sum = 0, i = 0;
  while (gclock() - start < dur_ns) {
    const uint64_t t0 = gclock();
    uint32_t v = 0;
    for (int b = 0; b < batches; ++b) v |= uint32_t(ld_relaxed_gpu(hot + ((i + b) * 32 + threadIdx.x) % 4096 * 32));
    v = __reduce_or_sync(~0u, v);
    const uint64_t t1 = gclock();
    if (v != 12345) {
      sum += t1 - t0;
      ++rounds;
    }
    i += batches;
  }
  if (threadIdx.x == 0) {
    acc[2] = sum;
    acc[3] = rounds;
    dyn[0] = 0;
  }
}

int main() {
  const uint64_t bytes = 1ull << 30;
  const uint32_t ntiles = uint32_t(bytes / kTileBytes);
  char *in, *out;
  uint64_t* hot;
  unsigned long long* acc;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&hot, 4096 * 256);
  cudaMalloc(&acc, 64);
  cudaMemset(in, 1, bytes);
  cudaMemset(hot, 0, 4096 * 256);
  CUtensorMap tin, tout;
  make_rows128_map(&tin, in, bytes / 128, kThreads);
  make_rows128_map(&tout, out, bytes / 128, kThreads);
  const uint32_t dyn = kTileBytes + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int qdyn = 200 * 1024;
  cudaFuncSetAttribute(quiet_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, qdyn);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int batches : {1, 2, 4, 8}) {
    for (int loaded = 0; loaded < 2; ++loaded) {
      cudaMemset(acc, 0, 64);
      cudaDeviceSynchronize();
      quiet_kernel<<<1, 32, qdyn, s2>>>(hot, acc, 3000000, batches);  // 3 ms
      if (loaded)
        for (int r = 0; r < 20; ++r) stream_kernel<<<ntiles, kThreads, dyn, s1>>>(tin, tout, hot, acc);
      cudaDeviceSynchronize();
      unsigned long long h[4];
      cudaMemcpy(h, acc, 32, cudaMemcpyDeviceToHost);
      printf("{\"batches\": %d, \"streaming\": %d, \"quiet_round_ns\": %.0f, \"quiet_rounds\": %llu, "
             "\"busy_sm_round_ns\": %.0f}\n",
             batches, loaded, h[3] ? double(h[2]) / h[3] : 0.0, h[3], h[1] ? double(h[0]) / h[1] : 0.0);
    }
  }
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
