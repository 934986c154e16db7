// context_bench.cu — CUB / cuBLAS on the same B200, as CONTEXT for the
// primitive layer's numbers (north star: "CUB/cuBLAS numbers are recorded as
// context only").  Not part of the product.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/context_bench tools/context_bench.cu -lcublas
// Prints one JSON object with algorithmic GB/s (same byte accounting as bench.py).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cub/cub.cuh>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void fill(float* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = float((i * 2654435761u) % 1000) * 1e-3f;
}

struct Sq {
  __host__ __device__ float operator()(float x) const { return x * x; }
};

template <class Fn>
float time_ms(Fn&& fn, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fn();
  cudaDeviceSynchronize();
  float best = 1e30f, sum = 0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    sum += ms;
    best = ms < best ? ms : best;
  }
  return sum / reps;
}

int main() {
  const size_t n30 = size_t(1) << 30, n28 = size_t(1) << 28;
  float *x, *y, *out;
  CK(cudaMalloc(&x, n30 * 4));
  CK(cudaMalloc(&y, n28 * 4));
  CK(cudaMalloc(&out, 64));
  fill<<<4096, 256>>>(x, n30);
  CK(cudaDeviceSynchronize());

  // DeviceReduce: sum of squares over 2^30 f32 (TransformReduce)
  void* tmp = nullptr;
  size_t tb = 0, tb2 = 0;
  auto it = cub::TransformInputIterator<float, Sq, float*>(x, Sq{});
  cub::DeviceReduce::Sum(nullptr, tb, it, out, n30);
  cub::DeviceScan::InclusiveSum(nullptr, tb2, x, y, n28);
  CK(cudaMalloc(&tmp, tb > tb2 ? tb : tb2));
  float ms_red = time_ms([&] { cub::DeviceReduce::Sum(tmp, tb, it, out, n30); });
  float ms_scan = time_ms([&] { cub::DeviceScan::InclusiveSum(tmp, tb2, x, y, n28); });
  float ms_escan = time_ms([&] { cub::DeviceScan::ExclusiveSum(tmp, tb2, x, y, n28); });

  // cuBLAS sgemv 16384^2, column-major A
  const int N = 16384;
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return 1;
  const float one = 1.f, zero = 0.f;
  float* xv = y;            // 16384 floats
  float* yv = y + N;        // 16384 floats
  float ms_n = time_ms([&] { cublasSgemv(h, CUBLAS_OP_N, N, N, &one, x, N, xv, 1, &zero, yv, 1); });
  float ms_t = time_ms([&] { cublasSgemv(h, CUBLAS_OP_T, N, N, &one, x, N, xv, 1, &zero, yv, 1); });

  auto gbs = [](double bytes, float ms) { return bytes / (ms * 1e-3) / 1e9; };
  std::printf(
      "{\"cub_reduce_sumsq_f32_2^30\": {\"ms\": %.4f, \"gbs\": %.1f}, "
      "\"cub_inclusive_sum_f32_2^28\": {\"ms\": %.4f, \"gbs\": %.1f}, "
      "\"cub_exclusive_sum_f32_2^28\": {\"ms\": %.4f, \"gbs\": %.1f}, "
      "\"cublas_sgemv_N_16384^2 (gemv, ref vecmat)\": {\"ms\": %.4f, \"gbs\": %.1f}, "
      "\"cublas_sgemv_T_16384^2 (gevm, ref matvec)\": {\"ms\": %.4f, \"gbs\": %.1f}}\n",
      ms_red, gbs(double(n30) * 4, ms_red), ms_scan, gbs(double(n28) * 8, ms_scan), ms_escan,
      gbs(double(n28) * 8, ms_escan), ms_n, gbs(double(N) * N * 4 + 2.0 * N * 4, ms_n), ms_t,
      gbs(double(N) * N * 4 + 2.0 * N * 4, ms_t));
  cublasDestroy(h);
  return 0;
}
