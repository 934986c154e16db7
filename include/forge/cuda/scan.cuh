// forge/cuda/scan.cuh — single-pass decoupled look-back scan for sm_100a.
//
// Reference: prim::scan (primitives.hpp:440-603).  Same protocol, re-designed
// for real hardware:
//   * tile = 256 threads x IT items (IT = 64 B / max(sizeof T, sizeof S), <= 16:
//     4096 f32, 2048 8-byte structs, 1024 16-byte structs); each thread loads
//     its IT contiguous items with 256-bit ld.global.nc.v8 (primitives.hpp:486-498
//     did a 16-wide vload per thread) and runs a register scan;
//   * tile ids come from an atomic ticket, not blockIdx.x (the VM admitted
//     blocks in id order, machine.cpp:767-776; CUDA does not guarantee that, so
//     a tile could otherwise spin on a predecessor that is not resident);
//   * tile status: every 32-bit chunk of the published carry travels in its own
//     64-bit word {status, chunk}; a reader accepts a state only when all words
//     carry the same status, so no fence and no separate flag byte are needed
//     (the reference used a relaxed aggregate store + release flag,
//     primitives.hpp:518-534, 568-575);
//   * status = (epoch << 2) | {1 PARTIAL, 2 PREFIX}; the epoch advances at the
//     end of every launch (the last tile to finish its look-back bumps it), so
//     stale states of earlier launches read as INVALID and the workspace needs
//     no fill_zero per launch (primitives.hpp:464-466);
//   * look-back: warp 0 polls 32 predecessors at once, finds the nearest PREFIX
//     with one ballot and folds the window with a log-step ORDER-PRESERVING
//     reduction (the reference folded the window serially with 32 shuffles,
//     primitives.hpp:561-563);
//   * the inter-tile carry chain runs in CarryTraits<S,Op>::C (f64 for the f32
//     sums), per-element work in S;
//   * optional carry_in (the exclusive prefix of earlier shards, sharded scan)
//     and total_out (the inclusive total) device operands.
#pragma once

#include "forge/cuda/reduce.cuh"

namespace forge::cuda {

constexpr int kScanThreads = 256;
constexpr uint32_t kPartial = 1, kPrefix = 2;

template <class C>
struct TileStateIO {
  static constexpr int SW = Words<C>::N;  // 32-bit chunks of the carry
  static constexpr int STRIDE = SW <= 1 ? 1 : SW <= 2 ? 2 : SW <= 4 ? 4 : SW <= 8 ? 8 : 16;

  static __device__ __forceinline__ void write(uint64_t* states, uint64_t tile, uint32_t epoch,
                                               uint32_t kind, const C& v) {
    Words<C> w = to_words(v);
    const uint64_t hi = uint64_t((epoch << 2) | kind) << 32;
    uint64_t* p = states + tile * STRIDE;
    if constexpr (STRIDE == 1) {
      st_relaxed_gpu(p, hi | w.w[0]);
    } else {
#pragma unroll
      for (int i = 0; i < STRIDE; i += 2) {
        const uint64_t a = hi | (i < SW ? w.w[i] : 0u);
        const uint64_t b = hi | (i + 1 < SW ? w.w[i + 1] : 0u);
        st_relaxed_gpu_v2(p + i, a, b);
      }
    }
  }

  // Returns the kind (0 = not yet valid for this epoch) and the value.
  static __device__ __forceinline__ uint32_t read(const uint64_t* states, uint64_t tile,
                                                  uint32_t epoch, C& v) {
    const uint64_t* p = states + tile * STRIDE;
    uint64_t raw[STRIDE];
    if constexpr (STRIDE == 1) {
      raw[0] = ld_relaxed_gpu(p);
    } else {
#pragma unroll
      for (int i = 0; i < STRIDE; i += 2) ld_relaxed_gpu_v2(p + i, raw[i], raw[i + 1]);
    }
    const uint32_t hi = uint32_t(raw[0] >> 32);
    bool same = true;
#pragma unroll
    for (int i = 1; i < SW; ++i) same &= uint32_t(raw[i] >> 32) == hi;
    const uint32_t kind = hi & 3u;
    if (!same || kind == 0 || (hi >> 2) != (epoch & 0x3fffffffu)) return 0;
    Words<C> w;
#pragma unroll
    for (int i = 0; i < SW; ++i) w.w[i] = uint32_t(raw[i]);
    v = from_words<C>(w);
    return kind;
  }
};

template <class T, class S, class F, class Op>
struct ScanArgs {
  const T* src;
  S* dst;
  uint64_t n;
  uint64_t src_stride, dst_stride;
  F f;
  Op op;
  S identity;          // exclusive output at index 0 when there is no carry-in
  const S* carry_in;   // nullable, device
  S* total_out;        // nullable, device
  uint64_t* states;    // [ntiles * STRIDE] 64-bit words
  uint32_t* ctrl;      // [0] ticket, [1] done counter, [2] epoch
  uint32_t ntiles;
};

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const ScanArgs<T, S, F, Op> a) {
  using CT = CarryTraits<S, Op>;
  using C = typename CT::C;
  using IO = TileStateIO<C>;
  constexpr int IT = scan_items<S>();
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  constexpr int NW = kScanThreads / kWarp;

  __shared__ uint32_t s_tile, s_epoch;
  __shared__ Opt<S> s_warp[NW];
  __shared__ Opt<S> s_carry;

  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  if (threadIdx.x == 0) {
    const uint32_t t = atom_add_relaxed_gpu(a.ctrl + 0, 1u);
    if (t == a.ntiles - 1) st_relaxed_gpu(a.ctrl + 0, 0u);  // all tiles claimed
    s_tile = t;
    s_epoch = ld_acquire_gpu(a.ctrl + 2);
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint32_t epoch = s_epoch;

  // ---- load + per-thread register scan (primitives.hpp:484-499)
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * IT;
  const uint64_t avail = base < a.n ? a.n - base : 0;
  const int count = avail >= uint64_t(IT) ? IT : int(avail);
  S regs[IT];
  if (count == IT && a.src_stride == 1 && is_aligned(a.src + base, items_align<T, IT>())) {
    T x[IT];
    load_items<T, IT>(a.src + base, x);
    regs[0] = a.f(x[0]);
#pragma unroll
    for (int k = 1; k < IT; ++k) regs[k] = a.op(regs[k - 1], a.f(x[k]));
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      if (k < count) {
        S v = a.f(a.src[(base + k) * a.src_stride]);
        regs[k] = k ? a.op(regs[k - 1], v) : v;
      }
    }
  }
  S last = regs[0];
#pragma unroll
  for (int k = 1; k < IT; ++k)
    if (k < count) last = regs[k];

  // ---- warp scan, then cross-warp scan through shared memory (:501-516)
  const Opt<S> incl = warp_scan_incl(a.op, Opt<S>{last, count > 0});
  if (lane == kWarp - 1) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    Opt<S> w = lane < NW ? s_warp[lane] : Opt<S>{S{}, false};
    w = warp_scan_incl(a.op, w);
    if (lane < NW) s_warp[lane] = w;
  }
  __syncthreads();
  const Opt<S> agg = s_warp[NW - 1];  // tile aggregate (a tile always holds >= 1 element)

  // ---- publish + decoupled look-back (:518-576)
  if (tile == 0) {
    if (threadIdx.x == 0) {
      Opt<S> cin = a.carry_in ? Opt<S>{*a.carry_in, true} : Opt<S>{S{}, false};
      C pre = CT::to_c(agg.v);
      if (cin.has) pre = CT::op(a.op, CT::to_c(cin.v), pre);
      IO::write(a.states, 0, epoch, kPrefix, pre);
      s_carry = cin;
      if (a.ntiles == 1 && a.total_out) *a.total_out = CT::to_s(pre);
    }
  } else if (warp == 0) {
    const C agg_c = CT::to_c(agg.v);
    if (lane == 0) IO::write(a.states, tile, epoch, kPartial, agg_c);
    auto cop = [&](const C& x, const C& y) { return CT::op(a.op, x, y); };
    Opt<C> carry{C{}, false};
    int64_t hi = int64_t(tile);
    for (;;) {
      const int64_t j = hi - 1 - int64_t(lane);
      C val{};
      uint32_t kind = 0;
      if (j >= 0) {
        while ((kind = IO::read(a.states, uint64_t(j), epoch, val)) == 0) {
        }
      }
      const unsigned pm = __ballot_sync(kFullMask, kind == kPrefix);
      const int pl = pm ? __ffs(int(pm)) - 1 : kWarp - 1;
      // Lanes 0..pl hold tiles hi-1 .. hi-1-pl (newest first); fold them with the
      // older (higher) lane on the LEFT of every combine.
      Opt<C> v{val, int(lane) <= pl && j >= 0};
#pragma unroll
      for (unsigned d = 1; d < kWarp; d <<= 1) {
        Opt<C> got{shfl_down(v.v, d), __shfl_down_sync(kFullMask, int(v.has), d) != 0};
        if (lane + d < kWarp) v = opt_combine(cop, got, v);
      }
      const Opt<C> window{shfl_idx(v.v, 0), __shfl_sync(kFullMask, int(v.has), 0) != 0};
      carry = opt_combine(cop, window, carry);
      if (pm) break;
      hi -= kWarp;
    }
    if (lane == 0) {
      const C inclusive_c = cop(carry.v, agg_c);
      IO::write(a.states, tile, epoch, kPrefix, inclusive_c);
      s_carry = Opt<S>{CT::to_s(carry.v), true};
      if (tile == a.ntiles - 1 && a.total_out) *a.total_out = CT::to_s(inclusive_c);
    }
  }
  __syncthreads();

  // This tile has finished reading predecessor states: count it; the last one
  // advances the epoch for the next launch and resets the counter.
  if (threadIdx.x == 0) {
    const uint32_t d = atom_add_acq_rel_gpu(a.ctrl + 1, 1u);
    if (d == a.ntiles - 1) {
      st_relaxed_gpu(a.ctrl + 1, 0u);
      st_relaxed_gpu(a.ctrl + 2, epoch + 1u);
    }
  }

  // ---- compose outputs in registers and store once (:579-600)
  const Opt<S> tile_ex = s_carry;
  const Opt<S> warp_ex = warp > 0 ? s_warp[warp - 1] : Opt<S>{S{}, false};
  Opt<S> lane_ex = shfl_up_opt(incl, 1);
  if (lane == 0) lane_ex.has = false;
  const Opt<S> pre = opt_combine(a.op, opt_combine(a.op, tile_ex, warp_ex), lane_ex);
  if (count == 0) return;
  S outs[IT];
  if constexpr (Inclusive) {
#pragma unroll
    for (int k = 0; k < IT; ++k) outs[k] = pre.has ? a.op(pre.v, regs[k]) : regs[k];
  } else {
    outs[0] = pre.has ? pre.v : a.identity;
#pragma unroll
    for (int k = 1; k < IT; ++k) outs[k] = pre.has ? a.op(pre.v, regs[k - 1]) : regs[k - 1];
  }
  if (count == IT && a.dst_stride == 1 && is_aligned(a.dst + base, items_align<S, IT>())) {
    store_items<S, IT>(a.dst + base, outs);
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k)
      if (k < count) a.dst[(base + k) * a.dst_stride] = outs[k];
  }
}

template <class T, class S, class Op>
struct ScanWs {
  using C = typename CarryTraits<S, Op>::C;
  static constexpr uint64_t kTile = uint64_t(kScanThreads) * scan_items<S>();
  static uint64_t tiles(uint64_t n) { return ceil_div(n, kTile); }
  static uint64_t bytes(uint64_t n) {
    return 256 + tiles(n) * TileStateIO<C>::STRIDE * sizeof(uint64_t);
  }
};

template <class T, class S, class F, class Op>
cudaError_t launch_scan(const T* src, uint64_t src_stride, S* dst, uint64_t dst_stride, uint64_t n,
                        bool inclusive, const F& f, const Op& op, const S& identity,
                        const S* carry_in, S* total_out, void* ws, cudaStream_t stream) {
  const uint64_t ntiles = ScanWs<T, S, Op>::tiles(n);
  if (ntiles == 0) return cudaSuccess;
  if (ntiles >= (1ull << 31)) return cudaErrorInvalidValue;
  ScanArgs<T, S, F, Op> a{src,      dst,       n,   src_stride, dst_stride,
                          f,        op,        identity, carry_in, total_out,
                          reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + 256),
                          static_cast<uint32_t*>(ws), uint32_t(ntiles)};
  if (inclusive)
    scan_kernel<T, S, F, Op, true><<<uint32_t(ntiles), kScanThreads, 0, stream>>>(a);
  else
    scan_kernel<T, S, F, Op, false><<<uint32_t(ntiles), kScanThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace forge::cuda
