// Probe of the sm_100a FMNMX semantics behind fmax_total / fmin_total
// (include/forge/algebra.hpp): NaN result bits and the sign of zero, both
// operand orders.  Development tool: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdint>
#include <cstdio>
__global__ void k(const float* a, const float* b, uint32_t* o, int n) {
  int i = threadIdx.x;
  if (i >= n) return;
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a[i]), "f"(b[i]));
  o[4 * i + 0] = __float_as_uint(r);
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a[i]), "f"(b[i]));
  o[4 * i + 1] = __float_as_uint(r);
  o[4 * i + 2] = __float_as_uint(fmaxf(a[i], b[i]));
  o[4 * i + 3] = __float_as_uint(fminf(a[i], b[i]));
}
int main() {
  const uint32_t A[] = {0x80000000u, 0x00000000u, 0x7fc00001u, 0x3f800000u, 0xffc00000u, 0x80000000u, 0x00000000u};
  const uint32_t B[] = {0x00000000u, 0x80000000u, 0x3f800000u, 0xffc00123u, 0x7f800000u, 0x80000000u, 0x00000000u};
  const int n = 7;
  float *da, *db;
  uint32_t* dout;
  cudaMalloc(&da, 64); cudaMalloc(&db, 64); cudaMalloc(&dout, 256);
  cudaMemcpy(da, A, 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(db, B, 4 * n, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(da, db, dout, n);
  uint32_t o[4 * 7];
  cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i)
    printf("a=%08x b=%08x  max.NaN=%08x min.NaN=%08x fmaxf=%08x fminf=%08x\n", A[i], B[i], o[4 * i], o[4 * i + 1],
           o[4 * i + 2], o[4 * i + 3]);
  return 0;
}
