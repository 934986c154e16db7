// forge/cuda/reduce.cuh — one-kernel mapreduce, the order-preserving reduce and
// the rank-order fold.
//
// Reference: prim::mapreduce (primitives.hpp:348-431).  The reference runs a
// fixed grid of 100 x 256 threads, a grid-stride scalar map, an ordered warp
// tree, a shared-memory cross-warp step, and block 0 spinning on the release
// flags of every other block (a forward-progress hazard on real hardware:
// block 0 may spin while blocks it waits for are not yet resident).
//
// sm_100a design:
//   * grid = #SM x resident CTAs (persistent style), 256 threads;
//   * 256-bit ld.global.nc.L1::no_allocate.v8 loads, UNROLL independent vectors
//     in flight per thread (128 B/thread, tens of MB chip-wide), NACC
//     independent per-thread accumulators (ILP and a shallower float chain);
//   * warp butterfly (mapreduce requires a commutative op) + smem cross-warp;
//   * inter-block: every block stores its partial and does ONE acq_rel ticket
//     RMW; the LAST block to arrive (not block 0) folds the partials in block
//     order.  No block ever waits for another, so there is no residency
//     assumption, the result is deterministic for a fixed grid, and the ticket
//     self-resets so the workspace needs no memset between launches.
#pragma once

#include "forge/cuda/device.cuh"

namespace forge::cuda {

constexpr int kReduceThreads = 256;

// Carry type for the sequential cross-tile chains (decoupled look-back carry,
// per-block tile accumulation of the ordered reduce).  Default: S itself.  An
// op opts into a wider carry by defining `using carry_traits = ...;` with the
// same static members (the menu's f32 sums carry in f64, the affine maps in
// Affine<double>); per-element work always stays in S.
//
// kWide = true additionally runs the WHOLE scan / ordered reduction in C (f32
// only at the boundary).  The menu uses it for product-type operators (affine
// maps, quaternions): every one of the n-1 multiplications of a product chain
// contributes its rounding error to the result whatever the tree shape, so an
// f32 evaluation drifts like sqrt(n)*eps (the reference's own f32 fold shows
// 1e-5 relative at n = 1e5); in f64 the result is within a few ulp of f32.
template <class S, class Op, class = void>
struct CarryTraits {
  using C = S;
  static constexpr bool kWide = false;
  static __device__ __forceinline__ C to_c(const S& s) { return s; }
  static __device__ __forceinline__ S to_s(const C& c) { return c; }
  static __device__ __forceinline__ C op(const Op& o, const C& a, const C& b) { return o(a, b); }
};

template <class S, class Op>
struct CarryTraits<S, Op, std::void_t<typename Op::carry_traits>> : Op::carry_traits {};

// kNarrowEmit (optional member of a wide carry policy): the scan's second pass
// — the per-element running prefixes that become the outputs — runs in S,
// started from the f64 exclusive prefix of the thread's row.  Aggregates and
// carries stay in C, so no rounding accumulates across tiles; each output
// carries only the ~(row length) f32 roundings of its own row.
template <class CT, class = void>
struct NarrowEmit : std::false_type {};
template <class CT>
struct NarrowEmit<CT, std::void_t<decltype(CT::kNarrowEmit)>> : std::bool_constant<CT::kNarrowEmit> {};

// Arithmetic of one scan / ordered reduction: values of type A live in
// registers and shared memory; lift() maps f's S result in, lower() maps out,
// to_c()/from_c() cross into the carry type.
template <class S, class Op, bool Wide = CarryTraits<S, Op>::kWide>
struct ScanMath {
  using CT = CarryTraits<S, Op>;
  using C = typename CT::C;
  using A = S;
  static constexpr bool kNarrowEmit = false;
  static __device__ __forceinline__ A lift(const S& s) { return s; }
  static __device__ __forceinline__ S lower(const A& a) { return a; }
  static __device__ __forceinline__ A comb(const Op& o, const A& x, const A& y) { return o(x, y); }
  static __device__ __forceinline__ C to_c(const A& a) { return CT::to_c(a); }
  static __device__ __forceinline__ A from_c(const C& c) { return CT::to_s(c); }
};

template <class S, class Op>
struct ScanMath<S, Op, true> {
  using CT = CarryTraits<S, Op>;
  using C = typename CT::C;
  using A = C;
  static constexpr bool kNarrowEmit = NarrowEmit<CT>::value;
  static __device__ __forceinline__ A lift(const S& s) { return CT::to_c(s); }
  static __device__ __forceinline__ S lower(const A& a) { return CT::to_s(a); }
  static __device__ __forceinline__ A comb(const Op& o, const A& x, const A& y) { return CT::op(o, x, y); }
  static __device__ __forceinline__ C to_c(const A& a) { return a; }
  static __device__ __forceinline__ A from_c(const C& c) { return c; }
};

template <class T>
constexpr int mr_vec_elems() {
  return (sizeof(T) <= 32 && (32 % sizeof(T)) == 0) ? int(32 / sizeof(T)) : 1;
}

// Block-wide commutative reduction; the result is valid in thread 0.
template <class S, class Op>
__device__ __forceinline__ Opt<S> block_reduce_comm(const Op& op, Opt<S> v, Opt<S>* smem) {
  v = warp_allreduce_comm(op, v);
  const unsigned warp = threadIdx.x / kWarp, lane = lane_id();
  const unsigned nwarps = blockDim.x / kWarp;
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    Opt<S> w = lane < nwarps ? smem[lane] : Opt<S>{S{}, false};
    w = warp_allreduce_comm(op, w);
    if (lane == 0) v = w;
  }
  __syncthreads();
  return v;
}

// Block-wide ORDERED reduction of one value per thread in thread order; the
// result is valid in thread 0.
template <class S, class Op>
__device__ __forceinline__ Opt<S> block_reduce_ordered(const Op& op, Opt<S> v, Opt<S>* smem) {
  v = warp_reduce_ordered(op, v);
  const unsigned warp = threadIdx.x / kWarp, lane = lane_id();
  const unsigned nwarps = blockDim.x / kWarp;
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    Opt<S> w = lane < nwarps ? smem[lane] : Opt<S>{S{}, false};
    w = warp_reduce_ordered(op, w);
    if (lane == 0) v = w;
  }
  __syncthreads();
  return v;
}

// ---------------------------------------------------------------------------
// mapreduce (commutative)

template <class T, class S, class F, class Op>
struct MapReduceArgs {
  const T* src;
  uint64_t n;
  uint64_t stride;  // in elements; 1 = contiguous
  F f;
  Op op;
  S* partials;         // [grid]
  uint32_t* part_has;  // [grid]
  uint32_t* ticket;    // self-resetting arrival counter
  S* out;              // device result (S)
  uint32_t* out_has;   // nullable
};

template <class T, class S, class F, class Op, int UNROLL>
__global__ void __launch_bounds__(kReduceThreads)
    mapreduce_kernel(const MapReduceArgs<T, S, F, Op> a) {
  constexpr int VE = mr_vec_elems<T>();
  constexpr int VB = VE * int(sizeof(T));
  constexpr int NACC = VE < 8 ? VE : 8;
  constexpr uint64_t kChunk = uint64_t(kReduceThreads) * UNROLL;
  __shared__ Opt<S> smem[kReduceThreads / kWarp];
  __shared__ bool s_last;

  const uint64_t gtid = uint64_t(blockIdx.x) * kReduceThreads + threadIdx.x;
  const uint64_t gsize = uint64_t(gridDim.x) * kReduceThreads;

  // One-byte inputs: T has 256 values, so the map is TABULATED per CTA (any f).
  // The table is replicated per lane (entry e of lane l at word 32e + l), so
  // every lookup of a warp hits 32 distinct banks.  Turns ~9 instructions per
  // element (unpack, convert, f) into ~3 for e.g. UnitFloat8 decode.
  constexpr bool kTab = sizeof(T) == 1 && sizeof(S) == 4;
  __shared__ uint32_t tab[kTab ? 256 * kWarp : 1];
  if constexpr (kTab) {
    for (int e = threadIdx.x; e < 256; e += kReduceThreads) {
      T x;
      const uint8_t b = uint8_t(e);
      memcpy(&x, &b, 1);
      const S y = a.f(x);
      uint32_t w;
      memcpy(&w, &y, 4);
#pragma unroll 8
      for (int l = 0; l < kWarp; ++l) tab[e * kWarp + l] = w;
    }
    __syncthreads();
  }
  const unsigned tab_lane = lane_id();
  auto fmap = [&](const T& x) -> S {
    if constexpr (kTab) {
      uint8_t b;
      memcpy(&b, &x, 1);
      const uint32_t w = tab[uint32_t(b) * kWarp + tab_lane];
      S y;
      memcpy(&y, &w, 4);
      return y;
    } else {
      return a.f(x);
    }
  };

  // Element k of a loaded vector.  Tabulated maps index the table straight from
  // the packed 32-bit words: byte b of word w scaled to its 128-byte table row
  // is one shift + one LOP3 ((t & 0x7F80) | lane*4), so a lookup costs shift,
  // LOP3, LDS (+ the op) instead of extract, multiply-add, LDS (UF8 sum at
  // 2^30: 4.85 -> 5.40 TB/s; a 64 KB table indexed by one PRMT per lookup
  // measured 5.03: 3 CTAs/SM instead of 4).
  const uint32_t tab_lane4 = lane_id() * 4u;
  auto fmap_vec = [&](const T (&xv)[VE], int k) -> S {
    if constexpr (kTab && VE % 4 == 0) {
      uint32_t w;
      memcpy(&w, reinterpret_cast<const unsigned char*>(xv) + (k & ~3), 4);
      const int b = k & 3;
      const uint32_t t = b == 0 ? (w << 7) : (w >> (8 * b - 7));
      const uint32_t off = (t & 0x7F80u) | tab_lane4;
      const uint32_t bits = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const unsigned char*>(tab) + off);
      S y;
      memcpy(&y, &bits, 4);
      return y;
    } else {
      return fmap(xv[k]);
    }
  };

  S acc[NACC];       // vector accumulators, valid iff vhas
  bool vhas = false;
  Opt<S> sacc{S{}, false};  // scalar (head / tail / strided) accumulator

  const bool vector_path =
      VE > 1 && a.stride == 1 && (reinterpret_cast<uintptr_t>(a.src) % sizeof(T)) == 0;
  if (vector_path) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(a.src);
    uint64_t head = ((VB - (addr % VB)) % VB) / sizeof(T);
    if (head > a.n) head = a.n;
    const uint64_t nvec = (a.n - head) / VE;
    const T* body = a.src + head;
    const uint64_t full_chunks = nvec / kChunk;
    uint64_t c = blockIdx.x;
    if (c < full_chunks) {
      T x[UNROLL][VE];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        load_items<T, VE>(body + (c * kChunk + u * kReduceThreads + threadIdx.x) * VE, x[u]);
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] = fmap_vec(x[0], k);
#pragma unroll
      for (int k = NACC; k < VE; ++k) acc[k % NACC] = a.op(acc[k % NACC], fmap_vec(x[0], k));
#pragma unroll
      for (int u = 1; u < UNROLL; ++u)
#pragma unroll
        for (int k = 0; k < VE; ++k) acc[k % NACC] = a.op(acc[k % NACC], fmap_vec(x[u], k));
      vhas = true;
      for (c += gridDim.x; c < full_chunks; c += gridDim.x) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          load_items<T, VE>(body + (c * kChunk + u * kReduceThreads + threadIdx.x) * VE, x[u]);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
#pragma unroll
          for (int k = 0; k < VE; ++k) acc[k % NACC] = a.op(acc[k % NACC], fmap_vec(x[u], k));
      }
    }
    // Leftover whole vectors, one per thread per pass.
    for (uint64_t v = full_chunks * kChunk + gtid; v < nvec; v += gsize) {
      T x[VE];
      load_items<T, VE>(body + v * VE, x);
      if (!vhas) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) acc[k] = fmap(x[k]);
#pragma unroll
        for (int k = NACC; k < VE; ++k) acc[k % NACC] = a.op(acc[k % NACC], fmap(x[k]));
        vhas = true;
      } else {
#pragma unroll
        for (int k = 0; k < VE; ++k) acc[k % NACC] = a.op(acc[k % NACC], fmap(x[k]));
      }
    }
    // Head and tail elements (fewer than 2*VE) go to the first threads.
    const uint64_t tail0 = head + nvec * VE;
    const uint64_t extra = head + (a.n - tail0);
    for (uint64_t e = gtid; e < extra; e += gsize) {
      const uint64_t i = e < head ? e : tail0 + (e - head);
      sacc = opt_combine(a.op, sacc, Opt<S>{fmap(a.src[i]), true});
    }
  } else {
    for (uint64_t i = gtid; i < a.n; i += gsize)
      sacc = opt_combine(a.op, sacc, Opt<S>{fmap(a.src[i * a.stride]), true});
  }

  Opt<S> mine = sacc;
  if (vhas) {
    S t = acc[0];
#pragma unroll
    for (int k = 1; k < NACC; ++k) t = a.op(t, acc[k]);
    mine = opt_combine(a.op, mine, Opt<S>{t, true});
  }
  Opt<S> blk = block_reduce_comm(a.op, mine, smem);

  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = blk.v;
    a.part_has[blockIdx.x] = blk.has ? 1u : 0u;
    const uint32_t t = atom_add_acq_rel_gpu(a.ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) st_relaxed_gpu(a.ticket, 0u);  // every block has arrived: reset for reuse
  }
  __syncthreads();
  if (!s_last) return;

  // Last block: fold the partials (deterministic tree for a fixed grid), with
  // kFoldBatch partial loads in flight per thread.
  constexpr int kFoldBatch = 8;
  Opt<S> v{S{}, false};
  for (uint32_t b0 = threadIdx.x; b0 < gridDim.x; b0 += kReduceThreads * kFoldBatch) {
    uint32_t hs[kFoldBatch];
    S ps[kFoldBatch];
#pragma unroll
    for (int q = 0; q < kFoldBatch; ++q) {
      const uint32_t b = b0 + uint32_t(q) * kReduceThreads;
      hs[q] = 0;
      if (b < gridDim.x) {
        hs[q] = ld_relaxed_gpu(a.part_has + b);
        ps[q] = ld_strong(a.partials + b);
      }
    }
#pragma unroll
    for (int q = 0; q < kFoldBatch; ++q)
      if (hs[q]) v = opt_combine(a.op, v, Opt<S>{ps[q], true});
  }
  Opt<S> total = block_reduce_comm(a.op, v, smem);
  if (threadIdx.x == 0) {
    *a.out = total.v;
    if (a.out_has) *a.out_has = total.has ? 1u : 0u;
  }
}

template <class T>
constexpr int mr_unroll() {
  return mr_vec_elems<T>() > 1 ? 4 : 8;
}

// Workspace layout (bytes) for mapreduce with `grid` blocks.
template <class S>
struct MapReduceWs {
  static constexpr uint64_t align(uint64_t v) { return (v + 255) & ~uint64_t(255); }
  static uint64_t bytes(uint32_t grid) {
    return align(sizeof(uint32_t) * 4) + align(uint64_t(grid) * sizeof(S)) +
           align(uint64_t(grid) * sizeof(uint32_t));
  }
  static void carve(void* ws, uint32_t grid, uint32_t*& ticket, S*& partials, uint32_t*& has) {
    char* p = static_cast<char*>(ws);
    ticket = reinterpret_cast<uint32_t*>(p);
    p += align(sizeof(uint32_t) * 4);
    partials = reinterpret_cast<S*>(p);
    p += align(uint64_t(grid) * sizeof(S));
    has = reinterpret_cast<uint32_t*>(p);
  }
};

// 4 CTAs per SM: measured best of 4..128 (more CTAs lengthen the last CTA's
// partial fold).  primitives.hpp's workspace bound assumes it.
inline uint32_t mapreduce_max_grid() { return uint32_t(device_props().sm_count) * 4; }

template <class T>
inline uint32_t mapreduce_grid(uint64_t n) {
  constexpr uint64_t per_block = uint64_t(kReduceThreads) * mr_vec_elems<T>() * mr_unroll<T>();
  uint64_t want = ceil_div(n, per_block);
  uint64_t cap = mapreduce_max_grid();
  return uint32_t(want < 1 ? 1 : (want > cap ? cap : want));
}

// ---------------------------------------------------------------------------
// Exact code sums.  A one-byte map that is affine in the code, f(c) = off +
// scale * c (e.g. UnitFloat8 decode = -1 + 2c/255, algebra.hpp:15-28), folded
// with a real-number sum: the result is n * off + scale * SUM(c), and SUM(c) is
// an exact integer — IDP4A (4 codes per instruction against 0x01010101) into
// 32-bit lane sums, flushed to 64 bits per pass.  One IDP4A per 4 input bytes
// instead of a table lookup + FADD per byte: the read roof at 1 byte per
// element.  The result is the real-number value of the sum rounded once; the
// tabulated path rounds each decoded term and the running sum instead
// (both within the f32 parity bar; the exact sum is the more accurate).
//
// A map opts in with `static constexpr bool kAffineCode = true;` plus
// kCodeOffset / kCodeScale; an op with `static constexpr bool kRealSum = true;`.
template <class F, class = void>
struct AffineCodeMap : std::false_type {};
template <class F>
struct AffineCodeMap<F, std::void_t<decltype(F::kAffineCode)>> : std::bool_constant<F::kAffineCode> {};
template <class Op, class = void>
struct RealSumOp : std::false_type {};
template <class Op>
struct RealSumOp<Op, std::void_t<decltype(Op::kRealSum)>> : std::bool_constant<Op::kRealSum> {};

template <class T, class S, class F, class Op>
constexpr bool code_sum_ok() {
  return sizeof(T) == 1 && (std::is_same_v<S, float> || std::is_same_v<S, double>) && AffineCodeMap<F>::value &&
         RealSumOp<Op>::value;
}

constexpr int kCodeSumUnroll = 4;  // 4 x 32 bytes in flight per thread

template <class S>
__global__ void __launch_bounds__(kReduceThreads)
    code_sum_kernel(const uint8_t* __restrict__ src, uint64_t n, double off, double scale,
                    unsigned long long* partials, uint32_t* ticket, S* out, uint32_t* out_has) {
  constexpr uint64_t kChunk = uint64_t(kReduceThreads) * kCodeSumUnroll;  // 32-byte vectors per chunk
  __shared__ unsigned long long smem[kReduceThreads / kWarp];
  __shared__ bool s_last;
  const uint64_t gtid = uint64_t(blockIdx.x) * kReduceThreads + threadIdx.x;
  const uint64_t gsize = uint64_t(gridDim.x) * kReduceThreads;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(src);
  uint64_t head = (32 - addr % 32) % 32;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 32;
  const uint8_t* body = src + head;
  unsigned long long total = 0;
  auto sum32 = [](const uint32_t (&w)[8], uint32_t acc) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = __dp4a(w[k], 0x01010101u, acc);
    return acc;
  };
  const uint64_t full = nvec / kChunk;
  for (uint64_t c = blockIdx.x; c < full; c += gridDim.x) {
    uint32_t w[kCodeSumUnroll][8];
#pragma unroll
    for (int u = 0; u < kCodeSumUnroll; ++u)
      load_items<uint32_t, 8>(reinterpret_cast<const uint32_t*>(body + (c * kChunk + u * kReduceThreads + threadIdx.x) * 32),
                              w[u]);
    uint32_t acc = 0;  // <= 4 * 8 * 1020: no overflow
#pragma unroll
    for (int u = 0; u < kCodeSumUnroll; ++u) acc = sum32(w[u], acc);
    total += acc;
  }
  for (uint64_t v = full * kChunk + gtid; v < nvec; v += gsize) {
    uint32_t w[8];
    load_items<uint32_t, 8>(reinterpret_cast<const uint32_t*>(body + v * 32), w);
    total += sum32(w, 0u);
  }
  const uint64_t tail0 = head + nvec * 32;
  const uint64_t extra = head + (n - tail0);
  for (uint64_t e = gtid; e < extra; e += gsize) total += src[e < head ? e : tail0 + (e - head)];

  // block sum, then the last block to arrive folds the partials
  auto block_sum = [&](unsigned long long v) {
#pragma unroll
    for (int d = kWarp / 2; d >= 1; d >>= 1) v += __shfl_xor_sync(kFullMask, v, d);
    if (lane_id() == 0) smem[threadIdx.x / kWarp] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
      for (int w = 0; w < kReduceThreads / kWarp; ++w) t += smem[w];
    __syncthreads();
    return t;
  };
  const unsigned long long blk = block_sum(total);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = blk;
    const uint32_t t = atom_add_acq_rel_gpu(ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) st_relaxed_gpu(ticket, 0u);
  }
  __syncthreads();
  if (!s_last) return;
  unsigned long long v = 0;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += kReduceThreads) v += ld_strong(partials + b);
  const unsigned long long codes = block_sum(v);
  if (threadIdx.x == 0) {
    *out = S(off * double(n) + scale * double(codes));
    if (out_has) *out_has = n > 0 ? 1u : 0u;
  }
}

template <class S>
cudaError_t launch_code_sum(const uint8_t* src, uint64_t n, double off, double scale, S* out_dev,
                            uint32_t* out_has_dev, void* ws, cudaStream_t stream) {
  const uint32_t grid = mapreduce_grid<uint32_t>(ceil_div(n, 4));
  uint32_t* ticket;
  S* parts_s;
  uint32_t* has;
  MapReduceWs<S>::carve(ws, mapreduce_max_grid(), ticket, parts_s, has);
  // 64-bit partials span the partial and flag areas (>= 8 bytes per block)
  static_assert(sizeof(S) >= 4, "code sums carve 8 bytes per block from S partials + flags");
  auto* parts = reinterpret_cast<unsigned long long*>(parts_s);
  if (const cudaError_t e = ws_claim(ws, kWsTagTicket, 256, stream, MapReduceWs<S>::bytes(mapreduce_max_grid()));
      e != cudaSuccess)
    return e;
  code_sum_kernel<S><<<grid, kReduceThreads, 0, stream>>>(src, n, off, scale, parts, ticket, out_dev, out_has_dev);
  return cudaGetLastError();
}

// Launch; `ws` holds MapReduceWs<S>::bytes(mapreduce_max_grid()) zero-initialised bytes.
template <class T, class S, class F, class Op>
cudaError_t launch_mapreduce(const T* src, uint64_t n, uint64_t stride, const F& f, const Op& op,
                             S* out_dev, uint32_t* out_has_dev, void* ws, cudaStream_t stream) {
  if constexpr (code_sum_ok<T, S, F, Op>()) {
    if (stride == 1 && n > 0)
      return launch_code_sum<S>(reinterpret_cast<const uint8_t*>(src), n, double(F::kCodeOffset),
                                double(F::kCodeScale), out_dev, out_has_dev, ws, stream);
  }
  const uint32_t grid = mapreduce_grid<T>(stride == 1 ? n : n * 4);
  MapReduceArgs<T, S, F, Op> a{src, n, stride, f, op, nullptr, nullptr, nullptr, out_dev, out_has_dev};
  MapReduceWs<S>::carve(ws, mapreduce_max_grid(), a.ticket, a.partials, a.part_has);
  if (const cudaError_t e = ws_claim(ws, kWsTagTicket, 256, stream, MapReduceWs<S>::bytes(mapreduce_max_grid()));
      e != cudaSuccess)
    return e;
  mapreduce_kernel<T, S, F, Op, mr_unroll<T>()><<<grid, kReduceThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Order-preserving reduce: any associative op.  Block b owns a contiguous run
// of tiles; inside a tile each thread folds ITEMS contiguous elements in order,
// then an ordered warp/block tree; tiles are folded in order into a C carry;
// the last block to arrive folds the block partials in block order.

// Items per thread of a scan tile: 64 bytes of S (16 f32, 8 eight-byte structs,
// 4 sixteen-byte structs).  Depends on S only so that a workspace sized for S
// fits every T.
template <class S>
constexpr int scan_items() {
  constexpr int it = 64 / int(sizeof(S));
  return it < 1 ? 1 : (it > 16 ? 16 : it);
}

template <class T, class S>
constexpr int tile_items() {
  constexpr int big = sizeof(T) > sizeof(S) ? int(sizeof(T)) : int(sizeof(S));
  constexpr int it = 64 / big;
  return it < 1 ? 1 : (it > 16 ? 16 : it);
}

template <class T, class S, class F, class Op, class C>
struct OrderedReduceArgs {
  const T* src;
  uint64_t n;
  uint64_t stride;
  F f;
  Op op;
  uint64_t tiles_per_block;
  C* partials;
  uint32_t* part_has;
  uint32_t* ticket;
  S* out;
  uint32_t* out_has;
};

template <class T, class S, class F, class Op>
__global__ void __launch_bounds__(kReduceThreads)
    reduce_ordered_kernel(const OrderedReduceArgs<T, S, F, Op, typename CarryTraits<S, Op>::C> a) {
  using M = ScanMath<S, Op>;
  using CT = typename M::CT;
  using C = typename CT::C;
  using A = typename M::A;
  constexpr int IT = tile_items<T, S>();
  constexpr uint64_t kTile = uint64_t(kReduceThreads) * IT;
  constexpr int NW = kReduceThreads / kWarp;
  constexpr int VE = mr_vec_elems<T>();          // one 32-byte vector per lane per step
  constexpr uint64_t kStep = uint64_t(kWarp) * VE;
  constexpr int U = sizeof(T) >= 8 ? 2 : 4;      // steps in flight per warp
  static_assert(kTile % kStep == 0, "block runs start on whole warp steps");
  __shared__ Opt<C> wsum[NW];
  __shared__ bool s_last;
  auto cop = [&](const C& x, const C& y) { return CT::op(a.op, x, y); };
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;

  // The block's contiguous run splits into NW contiguous warp runs.  A warp
  // folds its run IN ORDER one coalesced step (32 lanes x 32 bytes) at a
  // time, U steps in flight: each lane folds its VE elements in order, an
  // ordered warp reduction combines the lanes, lane 0 folds the step into the
  // warp's carry (type C).  Warp carries are folded in warp order at the end:
  // one __syncthreads per block (the tile-by-tile block reduction this
  // replaces synchronised twice per 4096 elements: 4.7 TB/s).
  const uint64_t ntiles = ceil_div(a.n, kTile);
  const uint64_t t0 = uint64_t(blockIdx.x) * a.tiles_per_block;
  const uint64_t t1 = t0 + a.tiles_per_block < ntiles ? t0 + a.tiles_per_block : ntiles;
  const uint64_t b0 = t0 * kTile, b1 = t1 * kTile < a.n ? t1 * kTile : a.n;
  const uint64_t nsteps = b1 > b0 ? (b1 - b0) / kStep : 0;
  const uint64_t s0 = nsteps * warp / NW, s1 = nsteps * (warp + 1) / NW;
  const bool vec_ok = VE > 1 && a.stride == 1 && is_aligned(a.src, 32);
  Opt<C> wacc{C{}, false};  // meaningful in lane 0
  auto fold_step = [&](const Opt<A>& lane_v) {
    const Opt<A> r = warp_reduce_ordered(aop, lane_v);
    if (lane == 0 && r.has) {
      const C rc = M::to_c(r.v);
      wacc = wacc.has ? Opt<C>{cop(wacc.v, rc), true} : Opt<C>{rc, true};
    }
  };
  if (vec_ok) {
    for (uint64_t st = s0; st < s1; st += U) {
      T x[U][VE];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (st + u < s1) load_items<T, VE>(a.src + b0 + (st + u) * kStep + uint64_t(lane) * VE, x[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (st + u < s1) {
          A v = M::lift(a.f(x[u][0]));
#pragma unroll
          for (int k = 1; k < VE; ++k) v = aop(v, M::lift(a.f(x[u][k])));
          fold_step(Opt<A>{v, true});
        }
      }
    }
  } else {
    for (uint64_t i0 = b0 + s0 * kStep; i0 < b0 + s1 * kStep; i0 += kWarp) {
      const uint64_t i = i0 + lane;
      fold_step(Opt<A>{i < b1 ? M::lift(a.f(a.src[i * a.stride])) : A{}, i < b1});
    }
  }
  if (warp == NW - 1) {  // the run's tail (< one step) belongs to the last warp
    for (uint64_t i0 = b0 + nsteps * kStep; i0 < b1; i0 += kWarp) {
      const uint64_t i = i0 + lane;
      fold_step(Opt<A>{i < b1 ? M::lift(a.f(a.src[i * a.stride])) : A{}, i < b1});
    }
  }
  if (lane == 0) wsum[warp] = wacc;
  __syncthreads();
  Opt<C> bacc{C{}, false};  // meaningful in thread 0
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NW; ++w)
      if (wsum[w].has) bacc = bacc.has ? Opt<C>{cop(bacc.v, wsum[w].v), true} : wsum[w];
  }
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = bacc.v;
    a.part_has[blockIdx.x] = bacc.has ? 1u : 0u;
    const uint32_t t = atom_add_acq_rel_gpu(a.ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) st_relaxed_gpu(a.ticket, 0u);
  }
  __syncthreads();
  if (!s_last) return;
  // Last block: warp 0 folds partials in block order.  Lane L owns a
  // contiguous range of blocks, then an ordered warp reduction.
  if (threadIdx.x >= kWarp) return;
  const uint32_t nb = gridDim.x;
  const uint32_t per = (nb + kWarp - 1) / kWarp;
  const uint32_t lo = threadIdx.x * per, hi = lo + per < nb ? lo + per : nb;
  Opt<C> v{C{}, false};
  for (uint32_t b = lo; b < hi; ++b) {
    if (ld_relaxed_gpu(a.part_has + b)) {
      C pb = ld_strong(a.partials + b);
      v = v.has ? Opt<C>{cop(v.v, pb), true} : Opt<C>{pb, true};
    }
  }
  v = warp_reduce_ordered(cop, v);
  if (threadIdx.x == 0) {
    *a.out = CT::to_s(v.v);
    if (a.out_has) *a.out_has = v.has ? 1u : 0u;
  }
}

template <class S, class Op>
struct OrderedReduceWs {
  using C = typename CarryTraits<S, Op>::C;
  static constexpr uint64_t align(uint64_t v) { return (v + 255) & ~uint64_t(255); }
  static uint64_t bytes(uint32_t grid) {
    return align(sizeof(uint32_t) * 4) + align(uint64_t(grid) * sizeof(C)) +
           align(uint64_t(grid) * sizeof(uint32_t));
  }
  static void carve(void* ws, uint32_t grid, uint32_t*& ticket, C*& partials, uint32_t*& has) {
    char* p = static_cast<char*>(ws);
    ticket = reinterpret_cast<uint32_t*>(p);
    p += align(sizeof(uint32_t) * 4);
    partials = reinterpret_cast<C*>(p);
    p += align(uint64_t(grid) * sizeof(C));
    has = reinterpret_cast<uint32_t*>(p);
  }
};

template <class T, class S, class F, class Op>
cudaError_t launch_reduce_ordered(const T* src, uint64_t n, uint64_t stride, const F& f,
                                  const Op& op, S* out_dev, uint32_t* out_has_dev, void* ws,
                                  cudaStream_t stream) {
  using C = typename CarryTraits<S, Op>::C;
  constexpr uint64_t kTile = uint64_t(kReduceThreads) * tile_items<T, S>();
  const uint64_t ntiles = ceil_div(n, kTile);
  const uint32_t cap = mapreduce_max_grid();
  uint64_t grid = ntiles < cap ? ntiles : cap;
  if (grid < 1) grid = 1;
  const uint64_t per = ceil_div(ntiles, grid);
  grid = ntiles ? ceil_div(ntiles, per) : 1;
  OrderedReduceArgs<T, S, F, Op, C> a{src, n, stride, f, op, per, nullptr, nullptr, nullptr, out_dev, out_has_dev};
  OrderedReduceWs<S, Op>::carve(ws, cap, a.ticket, a.partials, a.part_has);
  if (const cudaError_t e = ws_claim(ws, kWsTagTicket, 256, stream, OrderedReduceWs<S, Op>::bytes(cap));
      e != cudaSuccess)
    return e;
  reduce_ordered_kernel<T, S, F, Op><<<uint32_t(grid), kReduceThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fold of a short device array in index order (rank-order fold of the sharded
// exchange).  upto < 0: all `count` values; else values[0..upto).

template <class S, class Op>
__global__ void fold_kernel(const S* values, uint32_t count, int32_t upto, Op op, S* out,
                            int32_t* has_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint32_t m = upto < 0 ? count : (uint32_t(upto) < count ? uint32_t(upto) : count);
  Opt<S> v{S{}, false};
  for (uint32_t i = 0; i < m; ++i) v = opt_combine(op, v, Opt<S>{values[i], true});
  if (v.has) *out = v.v;
  if (has_out) *has_out = v.has ? 1 : 0;
}

template <class S, class Op>
cudaError_t launch_fold(const S* values, uint32_t count, int32_t upto, const Op& op, S* out,
                        int32_t* has_out, cudaStream_t stream) {
  fold_kernel<S, Op><<<1, 32, 0, stream>>>(values, count, upto, op, out, has_out);
  return cudaGetLastError();
}

}  // namespace forge::cuda
