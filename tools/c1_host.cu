// c1_host.cu — development probe: host cost per call of the pieces of
// forge_dev_scan at the C1 size (2^20 f32).  Links libforge.so.
//   nvcc -O2 -std=c++20 -gencode arch=compute_100a,code=sm_100a -I include -I paper_2603_18695_b200/csrc \
//        --expt-relaxed-constexpr --extended-lambda -o tools/c1_host tools/c1_host.cu \
//        -L paper_2603_18695_b200 -lforge -Xlinker -rpath,$PWD/paper_2603_18695_b200
#include <chrono>
#include <cstdio>

#include "forge.h"
#include "forge/cuda/tma.cuh"

using namespace forge::cuda;

struct Big {
  unsigned char b[160];
};
__global__ void empty_kernel(const Big a, const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2) {
  if (a.b[0] == 7 && threadIdx.x == 999) printf("x");
}
__global__ void tiny_kernel(int* p) {
  if (threadIdx.x == 999) *p = 1;
}

template <class F>
double per_call_us(F&& f, int k = 5000) {
  for (int i = 0; i < 100; ++i) f();
  cudaDeviceSynchronize();
  auto t = std::chrono::steady_clock::now();
  for (int i = 0; i < k; ++i) f();
  const double host = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count() / k;
  cudaDeviceSynchronize();
  return host;
}

int main() {
  const uint64_t n = 1 << 20;
  float *src, *dst;
  void* ws;
  uint64_t wsb = 0;
  cudaMalloc(&src, n * 4);
  cudaMalloc(&dst, n * 4);
  cudaMemset(src, 0, n * 4);
  forge_dev_workspace_bytes(FORGE_PRIM_SCAN, FORGE_OP_F32_SUM, n, 0, &wsb);
  cudaMalloc(&ws, wsb);
  cudaMemset(ws, 0, wsb);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  CUtensorMap m1, m2;
  make_rows128_map(&m1, src, n * 4 / 128, 256);
  make_rows128_map(&m2, dst, n * 4 / 128, 256);
  Big big{};
  int* p;
  cudaMalloc(&p, 4);
  printf("{\"forge_dev_scan_host_us\": %.2f, ", per_call_us([&] {
           forge_dev_scan(FORGE_OP_F32_SUM, 1, src, dst, n, nullptr, nullptr, ws, wsb, s);
         }));
  printf("\"launch_400B_params_us\": %.2f, ", per_call_us([&] { empty_kernel<<<128, 256, 0, s>>>(big, m1, m2); }));
  printf("\"launch_tiny_us\": %.2f, ", per_call_us([&] { tiny_kernel<<<128, 256, 0, s>>>(p); }));
  printf("\"tensor_map_lookup_us\": %.3f, ", per_call_us([&] { make_rows128_map(&m1, src, n * 4 / 128, 256); }, 100000));
  printf("\"cudaGetDevice_us\": %.3f, ", per_call_us([&] { int d; cudaGetDevice(&d); }, 100000));
  printf("\"cudaGetLastError_us\": %.3f}\n", per_call_us([&] { cudaGetLastError(); }, 100000));
  return 0;
}
