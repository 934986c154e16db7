// probe_gemv.cu — development probe (not product): gemv_kernel (ref vecmat,
// z = A x, column-major A) at 16384^2 f32 over (U columns per load group,
// register budget MinB CTAs/SM, software-pipelined loads) x CTAs per SM of the
// split plan.  Prints GB/s (algorithmic bytes / CUDA-event time, median of 15).
//   nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -I include -o tools/probe_gemv tools/probe_gemv.cu
#include <algorithm>
#include <cstdio>
#include <vector>

#include "forge/cuda/matrix.cuh"

using namespace forge::cuda;

struct Mul {
  __host__ __device__ float operator()(float a, float x) const { return a * x; }
};
struct Add {
  __host__ __device__ float operator()(float a, float b) const { return a + b; }
};

__global__ void fill(float* p, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = float(h & 0xffff) * (1.0f / 65536.0f) - 0.5f;
  }
}

static uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

template <int U, int MinB, bool Pipe>
static void run(const char* name, const float* A, const float* x, float* z, uint64_t n, uint64_t p, char* ws,
                int per_sm, std::vector<float>& ref, int sms) {
  constexpr int VE = gemv_vec_elems<float>();
  const uint64_t row_blocks = cdiv(n, uint64_t(kMatThreads) * VE);
  const uint64_t target = uint64_t(sms) * per_sm;
  uint64_t ks = row_blocks >= target ? 1 : cdiv(target, row_blocks);
  ks = std::min<uint64_t>(ks, cdiv(p, 16));
  uint64_t cps = cdiv(p, ks);
  ks = cdiv(p, cps);
  uint32_t gsize = uint32_t(ks);
  if (ks > 8) {
    gsize = 1;
    while (uint64_t(gsize) * gsize < ks) ++gsize;
  }
  const uint32_t groups = uint32_t(cdiv(ks, gsize));
  GemvArgs<float, float, Mul, Add> a{A, x, z, n, p, n, Mul{}, Add{}, uint32_t(ks), cps, uint32_t(row_blocks),
                                     true, nullptr, nullptr, gsize, groups, nullptr};
  a.tickets = reinterpret_cast<uint32_t*>(ws);
  cudaMemset(ws, 0, 1 << 20);
  a.partials = reinterpret_cast<float*>(ws + (1 << 20));
  a.gpartials = a.partials + ks * n;
  const uint32_t grid = uint32_t(row_blocks * ks);
  auto launch = [&] { gemv_kernel<float, float, Mul, Add, true, U, MinB, Pipe><<<grid, kMatThreads>>>(a); };
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ms;
  for (int i = 0; i < 15; ++i) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  std::vector<float> got(n);
  cudaMemcpy(got.data(), z, n * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  if (ref.empty()) ref = got;
  for (uint64_t i = 0; i < n; ++i) err = std::max(err, double(std::abs(got[i] - ref[i])));
  const double bytes = double(n) * p * 4 + double(p) * 4 + double(n) * 4;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gemv_kernel<float, float, Mul, Add, true, U, MinB, Pipe>);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_kernel<float, float, Mul, Add, true, U, MinB, Pipe>,
                                                kMatThreads, 0);
  printf("%-14s per_sm %2d ks %3llu grid %5u regs %3d occ %d  median %.4f ms  min %.4f  GB/s %.1f  maxdiff %.2e  %s\n",
         name, per_sm, (unsigned long long)ks, grid, fa.numRegs, occ, ms[7], ms[0], bytes / ms[7] / 1e6, err,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t n = 16384, p = 16384;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *A, *x, *z;
  char* ws;
  cudaMalloc(&A, n * p * 4);
  cudaMalloc(&x, p * 4);
  cudaMalloc(&z, n * 4);
  cudaMalloc(&ws, (1 << 20) + 300 * n * 4);
  fill<<<1184, 256>>>(A, n * p, 1);
  fill<<<64, 256>>>(x, p, 2);
  cudaDeviceSynchronize();
  std::vector<float> ref;
  for (int per_sm : {2, 3, 4, 6, 8, 12}) {
    run<4, 1, false>("U4", A, x, z, n, p, ws, per_sm, ref, sms);
    run<4, 4, false>("U4 mb4", A, x, z, n, p, ws, per_sm, ref, sms);
    run<8, 1, false>("U8", A, x, z, n, p, ws, per_sm, ref, sms);
    run<8, 2, false>("U8 mb2", A, x, z, n, p, ws, per_sm, ref, sms);
    run<2, 1, true>("U2 pipe", A, x, z, n, p, ws, per_sm, ref, sms);
    run<4, 1, true>("U4 pipe", A, x, z, n, p, ws, per_sm, ref, sms);
    run<4, 2, true>("U4 pipe mb2", A, x, z, n, p, ws, per_sm, ref, sms);
    run<2, 4, true>("U2 pipe mb4", A, x, z, n, p, ws, per_sm, ref, sms);
  }
  return 0;
}
