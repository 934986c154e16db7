// forge/cuda/device.cuh — sm_100a device building blocks for the primitive layer.
//
// Replaces the reference's portable intrinsics layer (KernelIntrinsics):
//   intr::shuffle / shuffle_up / shuffle_down  (intrinsics.hpp:138-175)
//       -> shfl_* : __shfl_sync over ceil(sizeof(T)/4) 32-bit words (padding is
//          moved harmlessly; CUDA's out-of-range convention equals the
//          reference's "keep own value", intrinsics.hpp:160-175)
//   intr::ordered_load / ordered_store        (intrinsics.hpp:100-109)
//       -> ld.acquire.gpu / st.release.gpu, plus relaxed.gpu strong accesses
//   intr::vload_n / vstore_n                  (intrinsics.hpp:218-254)
//       -> 256-bit ld.global.nc.L1::no_allocate.v8 / st.global.v8 (sm_100 only)
//   OptVal<S> / opt_combine                   (primitives.hpp:124-146)
//       -> Opt<S> (value + has flag kept in a predicate register)
//   warp_inclusive_scan / warp_reduce_ordered (primitives.hpp:153-170)
//       -> warp_scan_incl / warp_reduce_ordered (log-step, order-preserving)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#ifndef FORGE_HD
#define FORGE_HD __host__ __device__ __forceinline__
#endif

namespace forge::cuda {

constexpr int kWarp = 32;
constexpr unsigned kFullMask = 0xffffffffu;

// ---------------------------------------------------------------------------
// Optional accumulator (primitives.hpp:124-146): combine(a, b) folds b onto the
// right of a; an empty side yields the other.

template <class S>
struct Opt {
  S v;
  bool has;
};

template <class S, class Op>
__device__ __forceinline__ Opt<S> opt_combine(const Op& op, const Opt<S>& a, const Opt<S>& b) {
  if (!a.has) return b;
  if (!b.has) return a;
  return Opt<S>{op(a.v, b.v), true};
}

// ---------------------------------------------------------------------------
// Word-wise shuffles for any trivially copyable T.

template <class T>
struct Words {
  static constexpr int N = (int(sizeof(T)) + 3) / 4;
  uint32_t w[N];
};

template <class T>
__device__ __forceinline__ Words<T> to_words(const T& v) {
  static_assert(std::is_trivially_copyable_v<T>);
  Words<T> r;
  if constexpr (sizeof(T) % 4 != 0) r.w[Words<T>::N - 1] = 0;
  memcpy(r.w, &v, sizeof(T));
  return r;
}

template <class T>
__device__ __forceinline__ T from_words(const Words<T>& r) {
  T v;
  memcpy(&v, r.w, sizeof(T));
  return v;
}

template <class T>
__device__ __forceinline__ T shfl_idx(const T& v, int src, unsigned mask = kFullMask) {
  Words<T> w = to_words(v);
#pragma unroll
  for (int i = 0; i < Words<T>::N; ++i) w.w[i] = __shfl_sync(mask, w.w[i], src);
  return from_words<T>(w);
}

template <class T>
__device__ __forceinline__ T shfl_up(const T& v, unsigned delta, unsigned mask = kFullMask) {
  Words<T> w = to_words(v);
#pragma unroll
  for (int i = 0; i < Words<T>::N; ++i) w.w[i] = __shfl_up_sync(mask, w.w[i], delta);
  return from_words<T>(w);
}

template <class T>
__device__ __forceinline__ T shfl_down(const T& v, unsigned delta, unsigned mask = kFullMask) {
  Words<T> w = to_words(v);
#pragma unroll
  for (int i = 0; i < Words<T>::N; ++i) w.w[i] = __shfl_down_sync(mask, w.w[i], delta);
  return from_words<T>(w);
}

template <class T>
__device__ __forceinline__ T shfl_xor(const T& v, unsigned lane_mask) {
  Words<T> w = to_words(v);
#pragma unroll
  for (int i = 0; i < Words<T>::N; ++i) w.w[i] = __shfl_xor_sync(kFullMask, w.w[i], lane_mask);
  return from_words<T>(w);
}

template <class S>
__device__ __forceinline__ Opt<S> shfl_up_opt(const Opt<S>& v, unsigned d) {
  return Opt<S>{shfl_up(v.v, d), __shfl_up_sync(kFullMask, (int)v.has, d) != 0};
}
template <class S>
__device__ __forceinline__ Opt<S> shfl_down_opt(const Opt<S>& v, unsigned d) {
  return Opt<S>{shfl_down(v.v, d), __shfl_down_sync(kFullMask, (int)v.has, d) != 0};
}
template <class S>
__device__ __forceinline__ Opt<S> shfl_idx_opt(const Opt<S>& v, int src) {
  return Opt<S>{shfl_idx(v.v, src), __shfl_sync(kFullMask, (int)v.has, src) != 0};
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & (kWarp - 1); }

// Inclusive warp scan in lane order (Kogge-Stone, primitives.hpp:153-160):
// lane L ends with the fold of lanes 0..L.  Safe for non-commutative ops.
template <class S, class Op>
__device__ __forceinline__ Opt<S> warp_scan_incl(const Op& op, Opt<S> v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (unsigned d = 1; d < kWarp; d <<= 1) {
    Opt<S> got = shfl_up_opt(v, d);
    if (lane >= d) v = opt_combine(op, got, v);
  }
  return v;
}

// Ordered reduction (primitives.hpp:163-170): lane 0 ends with lane0 op lane1
// op ... op lane31, operands never reordered.
template <class S, class Op>
__device__ __forceinline__ Opt<S> warp_reduce_ordered(const Op& op, Opt<S> v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (unsigned d = 1; d < kWarp; d <<= 1) {
    Opt<S> got = shfl_down_opt(v, d);
    if (lane + d < kWarp) v = opt_combine(op, v, got);
  }
  return v;
}

// Butterfly reduction for commutative ops: every lane ends with the total.
template <class S, class Op>
__device__ __forceinline__ Opt<S> warp_allreduce_comm(const Op& op, Opt<S> v) {
#pragma unroll
  for (unsigned d = kWarp / 2; d >= 1; d >>= 1) {
    Opt<S> got{shfl_xor(v.v, d), __shfl_xor_sync(kFullMask, (int)v.has, d) != 0};
    v = opt_combine(op, v, got);
  }
  return v;
}

// ---------------------------------------------------------------------------
// Ordered / strong global accesses.

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void ld_relaxed_gpu_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];"
               : "=l"(a), "=l"(b)
               : "l"(p)
               : "memory");
}
// 256-bit relaxed load (LDG.E.ENL2.256.STRONG.GPU): a 32-byte-aligned group
// of tile states in one L2 sector request; each 64-bit element is
// single-copy atomic on its own.
__device__ __forceinline__ void ld_relaxed_gpu_v4(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                                  uint64_t& d) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_v2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// Ticket RMW with acquire+release semantics at GPU scope.
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint64_t atom_add_acq_rel_gpu(uint64_t* p, uint64_t v) {
  uint64_t r;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint64_t atom_add_relaxed_gpu(uint64_t* p, uint64_t v) {
  uint64_t r;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t atom_add_relaxed_gpu(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}

// Strong (L1-bypassing) load of an arbitrary trivially-copyable value, word by word.
template <class T>
__device__ __forceinline__ T ld_strong(const T* p) {
  if constexpr (sizeof(T) % 4 == 0 && alignof(T) >= 4) {
    Words<T> w;
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < Words<T>::N; ++i) w.w[i] = ld_relaxed_gpu(q + i);
    return from_words<T>(w);
  } else {
    return *static_cast<const volatile T*>(p);
  }
}

// ---------------------------------------------------------------------------
// Vector memory access.  V bytes per access, V in {1,2,4,8,16,32}.

template <int V>
struct VecBytes {
  uint32_t w[V / 4 > 0 ? V / 4 : 1];
};

template <int V>
__device__ __forceinline__ void ld_stream(const void* p, void* out) {
  uint32_t* r = static_cast<uint32_t*>(out);
  if constexpr (V == 32) {
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p));
  } else if constexpr (V == 16) {
    asm("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
        : "l"(p));
  } else if constexpr (V == 8) {
    asm("ld.global.nc.L1::no_allocate.v2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "l"(p));
  } else if constexpr (V == 4) {
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r[0]) : "l"(p));
  } else if constexpr (V == 2) {
    unsigned short h;
    asm("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(h) : "l"(p));
    memcpy(out, &h, 2);
  } else {
    static_assert(V == 1);
    *static_cast<unsigned char*>(out) = __ldg(static_cast<const unsigned char*>(p));
  }
}

// Cached read-only load (for re-used operands such as the matvec vector).
template <int V>
__device__ __forceinline__ void ld_cached(const void* p, void* out) {
  uint32_t* r = static_cast<uint32_t*>(out);
  if constexpr (V == 32) {
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p));
  } else if constexpr (V == 16) {
    asm("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
        : "l"(p));
  } else if constexpr (V == 8) {
    asm("ld.global.nc.v2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "l"(p));
  } else if constexpr (V == 4) {
    asm("ld.global.nc.b32 %0, [%1];" : "=r"(r[0]) : "l"(p));
  } else {
    ld_stream<V>(p, out);
  }
}

template <int V>
__device__ __forceinline__ void st_vec(void* p, const void* in) {
  const uint32_t* r = static_cast<const uint32_t*>(in);
  if constexpr (V == 32) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  } else if constexpr (V == 16) {
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
  } else if constexpr (V == 8) {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(r[0]), "r"(r[1]) : "memory");
  } else if constexpr (V == 4) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(r[0]) : "memory");
  } else if constexpr (V == 2) {
    *static_cast<unsigned short*>(p) = *static_cast<const unsigned short*>(in);
  } else {
    *static_cast<unsigned char*>(p) = *static_cast<const unsigned char*>(in);
  }
}

// Largest power-of-two access width (<= 32 bytes) that divides `bytes`.
constexpr int vec_width(int bytes) {
  return bytes % 32 == 0 ? 32 : bytes % 16 == 0 ? 16 : bytes % 8 == 0 ? 8 : bytes % 4 == 0 ? 4
         : bytes % 2 == 0                      ? 2
                                               : 1;
}

// Loads N contiguous T (N * sizeof(T) bytes) with the widest aligned accesses;
// the caller guarantees `p` is aligned to vec_width(N * sizeof(T)).
template <class T, int N, bool Stream = true>
__device__ __forceinline__ void load_items(const T* p, T (&out)[N]) {
  constexpr int kBytes = N * int(sizeof(T));
  constexpr int kV = vec_width(kBytes);
  alignas(16) unsigned char buf[kBytes];
  const unsigned char* src = reinterpret_cast<const unsigned char*>(p);
#pragma unroll
  for (int b = 0; b < kBytes; b += kV) {
    if constexpr (Stream) ld_stream<kV>(src + b, buf + b);
    else ld_cached<kV>(src + b, buf + b);
  }
  memcpy(out, buf, kBytes);
}

template <class T, int N>
__device__ __forceinline__ void store_items(T* p, const T (&in)[N]) {
  constexpr int kBytes = N * int(sizeof(T));
  constexpr int kV = vec_width(kBytes);
  alignas(16) unsigned char buf[kBytes];
  memcpy(buf, in, kBytes);
  unsigned char* dst = reinterpret_cast<unsigned char*>(p);
#pragma unroll
  for (int b = 0; b < kBytes; b += kV) st_vec<kV>(dst + b, buf + b);
}

template <class T, int N>
constexpr int items_align() {
  return vec_width(N * int(sizeof(T)));
}

__host__ __device__ __forceinline__ bool is_aligned(const void* p, int a) {
  return (reinterpret_cast<uintptr_t>(p) & uintptr_t(a - 1)) == 0;
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copies (cp.async.bulk, Hopper+/Blackwell async proxy).

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
// Makes mbarrier initialisation visible to the async proxy (TMA).
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D bulk copy global -> shared, completion signalled on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_addr(p)));
  return v;
}

// ---------------------------------------------------------------------------
// Host-side launch helpers.

// Development / experiment knobs.  Only builds compiled with -DFORGE_DEV
// (`make DEV=1` -> libforge_dev.so) read them from the environment; the
// product library uses the tuned defaults and never calls getenv.
#ifdef FORGE_DEV
inline uint32_t dev_knob(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return e ? uint32_t(std::strtoul(e, nullptr, 10)) : dflt;
}
#else
constexpr uint32_t dev_knob(const char*, uint32_t dflt) { return dflt; }
#endif

struct DeviceProps {
  int sm_count = 148;
  int device = -1;
};

inline const DeviceProps& device_props() {
  static thread_local DeviceProps cache;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cache.device != dev) {
    cache.device = dev;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      cache.sm_count = sms;
  }
  return cache;
}

// Workspace layout registry (defined in libforge.so, csrc/machine.cu).  Every
// primitive's kernels keep their own invariants on the workspace bytes they
// use (arrival tickets at zero, scan epochs), restored by the kernels
// themselves at the end of every launch — but two primitives (or two shapes of
// the matrix kernels) place tickets and partials at different offsets, so a
// workspace passed to another layout would see the previous layout's partials
// as tickets.  Each launch therefore claims `ws` for its layout `tag`; when
// the pointer was last used with another tag (or is unknown), the first
// `zero_bytes` bytes are zeroed on `stream` before the kernel (the reference
// zero-fills its flags on every launch, primitives.hpp:374, :464-466, :759);
// with the same tag, only bytes beyond the extent zeroed before.  A claim
// also invalidates every other claim whose bytes it overlaps (a sub-workspace
// at an offset, e.g. the lagged scan's tail launch), so those re-zero on
// their next use.
// `extent_bytes` (>= zero_bytes; 0 = zero_bytes): every byte of ws the launch
// may write, for the overlap invalidation.
cudaError_t ws_claim(void* ws, uint64_t tag, uint64_t zero_bytes, cudaStream_t stream, uint64_t extent_bytes = 0);

// Layout tags.
constexpr uint64_t kWsTagTicket = 1;  // mapreduce / ordered reduce: ticket word at offset 0
constexpr uint64_t kWsTagScan = 2;    // scan: control block + epoch-tagged tile states
constexpr uint64_t kWsTagScanLag = 3; // lagged scan: control block + tile aggregates + group states
constexpr uint64_t kWsTagScanCyclic = 4;  // cross-GPU cyclic scan: ticket + per-local-tile states
inline uint64_t ws_tag(uint64_t kind, uint64_t a, uint64_t b = 0) { return kind | (a << 8) | (b << 40); }

__host__ __device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

}  // namespace forge::cuda
