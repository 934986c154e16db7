// test_shuffle.cu — SPEC.md acceptance #7 ("composite shuffle: fieldwise-oracle
// equality for 100 random descriptors x 100 random values x all source lanes,
// including the MisalignedStruct test type") on the sm_100a shuffles of
// forge/cuda/device.cuh, the B200 replacement of intr::shuffle / shuffle_up /
// shuffle_down (reference intrinsics.hpp:138-175).
//
// Each descriptor is generated as a literal (bitstype.hpp syntax) and parsed;
// values are random bytes (padding included).  A kernel instantiated for the
// descriptor's byte size moves the values with shfl_idx from every source lane,
// and with shfl_up / shfl_down by every delta (out-of-range sources keep their
// own value, intrinsics.hpp:160-175).  The host compares every result with the
// expected source value on the descriptor's data bytes (value_bytes_equal:
// padding is not part of a value).  Built by `make cpptests`, run by
// tests/test_gpu_cpp.py.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "forge/algebra.hpp"
#include "forge/bitstype.hpp"
#include "forge/cuda/device.cuh"
#include "forge/intrinsics.hpp"

using namespace forge;

namespace {

constexpr int kMaxBytes = 64;
constexpr int kWarps = 4;  // 128 lanes: 100 random values + 28 more
constexpr int kLanes = kWarps * 32;

template <int N>
struct Blob {
  unsigned char b[N];
};

// out_idx[w][src][lane], out_up[w][d][lane], out_down[w][d][lane]
template <int N>
__global__ void shuffle_kernel(const Blob<N>* in, Blob<N>* out_idx, Blob<N>* out_up, Blob<N>* out_down) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Blob<N> v = in[threadIdx.x];
  for (int src = 0; src < 32; ++src) out_idx[(w * 32 + src) * 32 + lane] = cuda::shfl_idx(v, src);
  for (int d = 0; d < 32; ++d) {
    out_up[(w * 32 + d) * 32 + lane] = cuda::shfl_up(v, unsigned(d));
    out_down[(w * 32 + d) * 32 + lane] = cuda::shfl_down(v, unsigned(d));
  }
}

struct Result {
  long checks = 0, bad = 0;
};

template <int N>
void run_size(const TypeDescriptor& desc, std::mt19937_64& rng, Result& res) {
  static_assert(N >= 1 && N <= kMaxBytes);
  std::vector<Blob<N>> in(kLanes);
  for (auto& v : in)
    for (auto& c : v.b) c = static_cast<unsigned char>(rng());
  Blob<N>*d_in, *d_idx, *d_up, *d_down;
  const size_t outn = size_t(kWarps) * 32 * 32;
  cudaMalloc(&d_in, sizeof(Blob<N>) * kLanes);
  cudaMalloc(&d_idx, sizeof(Blob<N>) * outn);
  cudaMalloc(&d_up, sizeof(Blob<N>) * outn);
  cudaMalloc(&d_down, sizeof(Blob<N>) * outn);
  cudaMemcpy(d_in, in.data(), sizeof(Blob<N>) * kLanes, cudaMemcpyHostToDevice);
  shuffle_kernel<N><<<1, kLanes>>>(d_in, d_idx, d_up, d_down);
  std::vector<Blob<N>> idx(outn), up(outn), down(outn);
  cudaMemcpy(idx.data(), d_idx, sizeof(Blob<N>) * outn, cudaMemcpyDeviceToHost);
  cudaMemcpy(up.data(), d_up, sizeof(Blob<N>) * outn, cudaMemcpyDeviceToHost);
  cudaMemcpy(down.data(), d_down, sizeof(Blob<N>) * outn, cudaMemcpyDeviceToHost);
  cudaFree(d_in);
  cudaFree(d_idx);
  cudaFree(d_up);
  cudaFree(d_down);
  auto same = [&](const Blob<N>& a, const Blob<N>& b) {
    ++res.checks;
    const bool ok = value_bytes_equal(desc, std::as_bytes(std::span(a.b, N)), std::as_bytes(std::span(b.b, N)));
    if (!ok) ++res.bad;
    return ok;
  };
  for (int w = 0; w < kWarps; ++w)
    for (int k = 0; k < 32; ++k)
      for (int lane = 0; lane < 32; ++lane) {
        const size_t o = (size_t(w) * 32 + k) * 32 + lane;
        same(idx[o], in[w * 32 + k]);                                    // shuffle from source lane k
        same(up[o], in[w * 32 + (lane >= k ? lane - k : lane)]);         // shuffle_up by k
        same(down[o], in[w * 32 + (lane + k < 32 ? lane + k : lane)]);   // shuffle_down by k
      }
}

template <int N = 1>
void dispatch(int size, const TypeDescriptor& desc, std::mt19937_64& rng, Result& res) {
  if constexpr (N <= kMaxBytes) {
    if (size == N) return run_size<N>(desc, rng, res);
    dispatch<N + 1>(size, desc, rng, res);
  }
}

// Random descriptor literal: primitives, tuples (natural alignment), structs
// (explicit offsets, padding, declared size), nested; total size <= 64.
std::string random_literal(std::mt19937_64& rng, int depth) {
  static const char* prims[] = {"u8", "u16", "u32", "u64", "f32", "f64"};
  const int kind = depth >= 2 ? 0 : int(rng() % 3);
  if (kind == 0) return prims[rng() % 6];
  const int n = 1 + int(rng() % 4);
  if (kind == 1) {
    std::string s = "tuple(";
    for (int i = 0; i < n; ++i) s += (i ? "," : "") + random_literal(rng, depth + 1);
    return s + ")";
  }
  // struct: place fields at aligned offsets with random gaps
  std::string s = "struct(";
  uint32_t off = 0, maxalign = 1;
  for (int i = 0; i < n; ++i) {
    const std::string f = random_literal(rng, depth + 1);
    const TypeDescriptor d = parse_descriptor(f);
    off += uint32_t(rng() % 3) * d.alignment();  // padding gap
    off = (off + d.alignment() - 1) / d.alignment() * d.alignment();
    s += (i ? "," : "") + f + "@" + std::to_string(off);
    off += d.size();
    maxalign = d.alignment() > maxalign ? d.alignment() : maxalign;
  }
  const uint32_t size = (off + uint32_t(rng() % 2) * maxalign + maxalign - 1) / maxalign * maxalign;
  return s + "; size=" + std::to_string(size) + ")";
}

}  // namespace

int main() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    std::printf("no CUDA device\n");
    return 2;
  }
  std::mt19937_64 rng(0x5EED0007);
  Result res;
  int descriptors = 0, misaligned = 0;
  // the reference's padding test type first (algebra.hpp:75-80)
  std::vector<TypeDescriptor> descs = {intr::descriptor_of<alg::MisalignedStruct>()};
  while (descs.size() < 100) {
    const TypeDescriptor d = parse_descriptor(random_literal(rng, 0));
    if (d.size() >= 1 && d.size() <= uint32_t(kMaxBytes)) descs.push_back(d);
  }
  for (const TypeDescriptor& d : descs) {
    const long before = res.bad;
    dispatch(int(d.size()), d, rng, res);
    ++descriptors;
    if (d == intr::descriptor_of<alg::MisalignedStruct>()) ++misaligned;
    if (res.bad != before) std::printf("FAIL descriptor %s: %ld mismatches\n", to_string(d).c_str(), res.bad - before);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  const bool ok = res.bad == 0 && e == cudaSuccess && descriptors == 100 && misaligned >= 1;
  std::printf("%s: %d descriptors (MisalignedStruct included: %d), %ld lane checks, %ld mismatches, cuda=%s\n",
              ok ? "PASS" : "FAIL", descriptors, misaligned, res.checks, res.bad, cudaGetErrorString(e));
  return ok ? 0 : 1;
}
