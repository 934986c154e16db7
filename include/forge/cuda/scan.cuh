// forge/cuda/scan.cuh — single-pass decoupled look-back scan for sm_100a.
//
// Reference: prim::scan (primitives.hpp:440-603).  Same protocol (tile
// aggregate published as PARTIAL, look-back over predecessors until a PREFIX,
// own PREFIX published, outputs composed in registers and stored once),
// re-designed for real hardware:
//   * tile = 256 threads x IT items, IT = 64 B / sizeof(S) (<= 16): 4096 f32,
//     2048 eight-byte structs, 1024 sixteen-byte structs;
//   * tile ids come from an atomic ticket, not blockIdx.x (the VM admitted
//     blocks in id order, machine.cpp:767-776; CUDA guarantees no such order,
//     so a tile could otherwise spin on a predecessor that never becomes
//     resident);
//   * tile status: every 32-bit chunk of the published value travels in its
//     own 64-bit word {status, chunk}; a reader accepts a state only when all
//     words carry the same status, so no fence and no separate flag byte are
//     needed (the reference: relaxed aggregate store + release flag,
//     primitives.hpp:518-534, 568-575);
//   * status = (epoch << 2) | {1 PARTIAL, 2 PREFIX}; the last tile to finish
//     its look-back advances the epoch, so stale states of earlier launches read
//     as INVALID and the workspace needs no fill_zero per launch
//     (primitives.hpp:464-466);
//   * look-back: warp 0 polls 32 predecessors at once, finds the nearest PREFIX
//     with one ballot and folds the window with a log-step ORDER-PRESERVING
//     reduction (the reference folded it serially, primitives.hpp:561-563);
//   * inter-tile carries run in CarryTraits<S,Op>::C (f64 for the f32 sums);
//     product-type ops run entirely in C (ScanMath, reduce.cuh);
//   * optional carry_in (exclusive prefix of earlier shards) and total_out.
//
// Two kernels share the tile code:
//   scan_tma_kernel      contiguous 16-B-aligned input: PERSISTENT CTAs (grid =
//                        #SM x occupancy); each CTA claims tiles in ticket order
//                        and keeps STAGES future tiles in flight with 1-D TMA
//                        bulk copies (cp.async.bulk + mbarrier) into shared
//                        memory, so HBM reads overlap the look-back and the
//                        stores of the current tile.  Shared-memory reads use a
//                        per-thread chunk rotation that makes the 64-byte-per-
//                        thread blocked read conflict-free.
//   scan_kernel          everything else (strided views, unaligned bases):
//                        one tile per CTA, direct vector / scalar loads.
#pragma once

#include "forge/cuda/reduce.cuh"

namespace forge::cuda {

constexpr int kScanThreads = 256;
constexpr int kScanStages = 3;
constexpr uint32_t kPartial = 1, kPrefix = 2;
constexpr uint32_t kNoTile = 0xffffffffu;
constexpr int kLookbackPerThread = 4;  // max look-back polls per thread (window 256 * 4)
constexpr uint32_t kStateSlotWords = 32;  // 256-byte tile-state slots

template <class C>
struct TileStateIO {
  static constexpr int SW = Words<C>::N;  // 32-bit chunks of the carry
  static constexpr int STRIDE = SW <= 1 ? 1 : SW <= 2 ? 2 : SW <= 4 ? 4 : SW <= 8 ? 8 : 16;

  // `stride` (64-bit words per tile, >= STRIDE) spreads tile states over L2
  // slices: slices are selected at 256-byte granularity, and every CTA in
  // flight polls the states of the most recent tiles.
  static __device__ __forceinline__ void write(uint64_t* states, uint64_t tile, uint32_t stride,
                                               uint32_t epoch, uint32_t kind, const C& v) {
    Words<C> w = to_words(v);
    const uint64_t hi = uint64_t((epoch << 2) | kind) << 32;
    uint64_t* p = states + tile * stride;
    if constexpr (STRIDE == 1) {
      st_relaxed_gpu(p, hi | w.w[0]);
    } else {
#pragma unroll
      for (int i = 0; i < STRIDE; i += 2) {
        const uint64_t lo_word = hi | (i < SW ? w.w[i] : 0u);
        const uint64_t hi_word = hi | (i + 1 < SW ? w.w[i + 1] : 0u);
        st_relaxed_gpu_v2(p + i, lo_word, hi_word);
      }
    }
  }

  // Returns the kind (0 = not yet valid for this epoch) and the value.
  static __device__ __forceinline__ uint32_t read(const uint64_t* states, uint64_t tile,
                                                  uint32_t stride, uint32_t epoch, C& v) {
    const uint64_t* p = states + tile * stride;
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
  S identity;         // exclusive output at index 0 when there is no carry-in
  const S* carry_in;  // nullable, device
  S* total_out;       // nullable, device
  uint64_t* states;   // [ntiles * STRIDE] 64-bit words
  uint32_t* ctrl;     // [0] ticket, [2] epoch
  uint32_t ntiles;
  uint32_t state_stride;  // 64-bit words per tile state
  uint32_t lookback;      // look-back polls per consumer thread (0 = warp 0 only, window 32)
};

// The 256 consumer threads synchronise on named barrier 1, so a producer warp
// outside the barrier never stalls them (and vice versa).
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kScanThreads) : "memory");
}

// Per-CTA shared state of one tile.
template <class A, class C>
struct ScanShared {
  Opt<A> warp[kScanThreads / kWarp];
  Opt<A> carry;
  int first[kScanThreads / kWarp];  // look-back: nearest PREFIX per warp
  Opt<C> lb[kScanThreads / kWarp];  // look-back: per-warp window folds
};

template <class S, class Op>
using ScanSharedOf = ScanShared<typename ScanMath<S, Op>::A, typename ScanMath<S, Op>::C>;

// Everything after the items are in registers: register scan, block scan,
// publish + look-back, compose, store.  `raw` holds this thread's IT input
// items; `count` how many are valid.
template <class T, class S, class F, class Op, bool Inclusive, int IT>
__device__ __forceinline__ void scan_tile_body(const ScanArgs<T, S, F, Op>& a, uint64_t tile,
                                               uint32_t epoch, const T (&raw)[IT], int count,
                                               ScanSharedOf<S, Op>& sh) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  constexpr int NW = kScanThreads / kWarp;
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };

  // ---- per-thread register scan (primitives.hpp:484-499)
  A regs[IT];
#pragma unroll
  for (int k = 0; k < IT; ++k) {
    if (k < count) {
      const A v = M::lift(a.f(raw[k]));
      regs[k] = k ? aop(regs[k - 1], v) : v;
    }
  }
  A last = regs[0];
#pragma unroll
  for (int k = 1; k < IT; ++k)
    if (k < count) last = regs[k];

  // ---- warp scan, cross-warp scan through shared memory (:501-516)
  const Opt<A> incl = warp_scan_incl(aop, Opt<A>{last, count > 0});
  if (lane == kWarp - 1) sh.warp[warp] = incl;
  consumer_sync();
  if (warp == 0) {
    Opt<A> w = lane < NW ? sh.warp[lane] : Opt<A>{A{}, false};
    w = warp_scan_incl(aop, w);
    if (lane < NW) sh.warp[lane] = w;
  }
  consumer_sync();
  const Opt<A> agg = sh.warp[NW - 1];  // every tile holds >= 1 element

  // ---- publish + decoupled look-back (:518-576)
  if (tile == 0) {
    if (threadIdx.x == 0) {
      C pre = M::to_c(agg.v);
      Opt<A> cin{A{}, false};
      if (a.carry_in) {
        cin = Opt<A>{M::lift(*a.carry_in), true};
        pre = cop(M::to_c(cin.v), pre);
      }
      IO::write(a.states, 0, a.state_stride, epoch, kPrefix, pre);
      sh.carry = cin;
      if (a.ntiles == 1 && a.total_out) *a.total_out = M::CT::to_s(pre);
    }
  } else {
    // Block-wide look-back: each consumer thread polls kLookbackPerThread
    // consecutive predecessors, so one L2 round trip inspects 1024 tiles — more
    // than the tiles in flight on a B200 — and a tile finds a PREFIX in one
    // round.  (A single-warp window of 32 caps the PREFIX frontier at ~32 tiles
    // per round trip, ~1 TB/s at B200 latencies; measured in profiles/.)
    constexpr int LB = kLookbackPerThread;
    const C agg_c = M::to_c(agg.v);
    if (threadIdx.x == 0) IO::write(a.states, tile, a.state_stride, epoch, kPartial, agg_c);
    Opt<C> carry{C{}, false};  // meaningful in thread 0
    if (a.lookback == 0) {
      // Warp 0 alone: lanes poll the 32 nearest predecessors per round.
      if (warp == 0) {
        int64_t hi = int64_t(tile);
        for (;;) {
          const int64_t j = hi - 1 - int64_t(lane);
          C val{};
          uint32_t kind = 0;
          if (j >= 0) {
            while ((kind = IO::read(a.states, uint64_t(j), a.state_stride, epoch, val)) == 0) {
            }
          }
          const unsigned pm = __ballot_sync(kFullMask, kind == kPrefix);
          const int pl = pm ? __ffs(int(pm)) - 1 : kWarp - 1;
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
      }
    } else {
      const int lbn = int(a.lookback < uint32_t(LB) ? a.lookback : uint32_t(LB));
      const int WIN = kScanThreads * lbn;
      int64_t hi = int64_t(tile);
      for (;;) {
        C val[LB];
        uint32_t kind[LB];
        int first = WIN;
#pragma unroll
        for (int q = 0; q < LB; ++q) {
          kind[q] = 0;
          val[q] = C{};
          const int64_t j = hi - 1 - int64_t(threadIdx.x) * lbn - q;
          if (q < lbn && j >= 0) {
            while ((kind[q] = IO::read(a.states, uint64_t(j), a.state_stride, epoch, val[q])) == 0) {
            }
          }
          if (kind[q] == kPrefix && first == WIN) first = int(threadIdx.x) * lbn + q;
        }
        // nearest PREFIX over the block (position 0 = tile hi-1)
        const unsigned pm = __ballot_sync(kFullMask, first < WIN);
        const int wfirst = __shfl_sync(kFullMask, first, pm ? __ffs(int(pm)) - 1 : 0);
        if (lane == 0) sh.first[warp] = pm ? wfirst : WIN;
        consumer_sync();
        int pl = WIN;
#pragma unroll
        for (int w = 0; w < NW; ++w) pl = sh.first[w] < pl ? sh.first[w] : pl;
        const bool found = pl < WIN;
        // Fold positions 0..pl, older (larger position) always on the LEFT.
        Opt<C> v{C{}, false};
#pragma unroll
        for (int q = LB - 1; q >= 0; --q) {
          const int pos = int(threadIdx.x) * lbn + q;
          if (kind[q] != 0 && pos <= pl) v = opt_combine(cop, v, Opt<C>{val[q], true});
        }
#pragma unroll
        for (unsigned d = 1; d < kWarp; d <<= 1) {
          Opt<C> got{shfl_down(v.v, d), __shfl_down_sync(kFullMask, int(v.has), d) != 0};
          if (lane + d < kWarp) v = opt_combine(cop, got, v);
        }
        if (lane == 0) sh.lb[warp] = v;
        consumer_sync();
        if (threadIdx.x == 0) {
          Opt<C> window{C{}, false};
#pragma unroll
          for (int w = NW - 1; w >= 0; --w) window = opt_combine(cop, window, sh.lb[w]);
          carry = opt_combine(cop, window, carry);
        }
        if (found) break;
        hi -= WIN;
        consumer_sync();  // sh.first / sh.lb are rewritten by the next round
      }
    }
    if (threadIdx.x == 0) {
      const C inclusive_c = cop(carry.v, agg_c);
      IO::write(a.states, tile, a.state_stride, epoch, kPrefix, inclusive_c);
      sh.carry = Opt<A>{M::from_c(carry.v), true};
      if (tile == a.ntiles - 1 && a.total_out) *a.total_out = M::CT::to_s(inclusive_c);
    }
  }
  consumer_sync();

  // ---- compose outputs in registers and store once (:579-600)
  const Opt<A> tile_ex = sh.carry;
  const Opt<A> warp_ex = warp > 0 ? sh.warp[warp - 1] : Opt<A>{A{}, false};
  Opt<A> lane_ex = shfl_up_opt(incl, 1);
  if (lane == 0) lane_ex.has = false;
  const Opt<A> pre = opt_combine(aop, opt_combine(aop, tile_ex, warp_ex), lane_ex);
  if (count == 0) return;
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * IT;
  S outs[IT];
  if constexpr (Inclusive) {
#pragma unroll
    for (int k = 0; k < IT; ++k) outs[k] = M::lower(pre.has ? aop(pre.v, regs[k]) : regs[k]);
  } else {
    outs[0] = pre.has ? M::lower(pre.v) : a.identity;
#pragma unroll
    for (int k = 1; k < IT; ++k) outs[k] = M::lower(pre.has ? aop(pre.v, regs[k - 1]) : regs[k - 1]);
  }
  if (count == IT && a.dst_stride == 1 && is_aligned(a.dst + base, items_align<S, IT>())) {
    store_items<S, IT>(a.dst + base, outs);
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k)
      if (k < count) a.dst[(base + k) * a.dst_stride] = outs[k];
  }
}

template <class T, int IT>
__device__ __forceinline__ int load_tile_items_global(const T* src, uint64_t stride, uint64_t n,
                                                      uint64_t base, T (&raw)[IT]) {
  const uint64_t avail = base < n ? n - base : 0;
  const int count = avail >= uint64_t(IT) ? IT : int(avail);
  if (count == IT && stride == 1 && is_aligned(src + base, items_align<T, IT>())) {
    load_items<T, IT>(src + base, raw);
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k)
      if (k < count) raw[k] = src[(base + k) * stride];
  }
  return count;
}

// ---------------------------------------------------------------------------
// General path: one tile per CTA.

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const ScanArgs<T, S, F, Op> a) {
  using A = typename ScanMath<S, Op>::A;
  constexpr int IT = scan_items<S>();
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ ScanSharedOf<S, Op> sh;
  if (threadIdx.x == 0) {
    // Epoch first, then the acq_rel claim: every CTA's epoch read happens
    // before the last claim, whose owner may then advance the epoch for the
    // NEXT launch (this launch keeps using the value each CTA cached).
    s_epoch = ld_acquire_gpu(a.ctrl + 2);
    const uint32_t t = atom_add_acq_rel_gpu(a.ctrl + 0, 1u);
    if (t == a.ntiles - 1) {  // exactly ntiles claims: this is the last one
      st_relaxed_gpu(a.ctrl + 0, 0u);
      st_relaxed_gpu(a.ctrl + 2, s_epoch + 1u);
    }
    s_tile = t;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  T raw[IT];
  const int count =
      load_tile_items_global<T, IT>(a.src, a.src_stride, a.n, tile * kTile + uint64_t(threadIdx.x) * IT, raw);
  scan_tile_body<T, S, F, Op, Inclusive, IT>(a, tile, s_epoch, raw, count, sh);
}

// ---------------------------------------------------------------------------
// Persistent TMA-pipelined path (contiguous, 16-byte aligned input).

// Reads IT items (IT * sizeof(T) bytes) of one thread from shared memory.  For
// 64-byte rows the four 16-byte chunks are read in an order rotated by
// (tid >> 1) & 3 — each quarter-warp phase then touches 8 distinct 16-byte bank
// groups (conflict-free) — and put back in logical order with two conditional
// swap stages.
template <class T, int IT>
__device__ __forceinline__ void load_items_smem(const T* row, T (&out)[IT]) {
  constexpr int kBytes = IT * int(sizeof(T));
  const unsigned char* p = reinterpret_cast<const unsigned char*>(row);
  if constexpr (kBytes == 64) {
    const unsigned r = (threadIdx.x >> 1) & 3u;
    uint4 c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = lds128(p + 16 * (k ^ r));
    if (r & 1u) {
      uint4 t = c[0]; c[0] = c[1]; c[1] = t;
      t = c[2]; c[2] = c[3]; c[3] = t;
    }
    if (r & 2u) {
      uint4 t = c[0]; c[0] = c[2]; c[2] = t;
      t = c[1]; c[1] = c[3]; c[3] = t;
    }
    memcpy(out, c, 64);
  } else if constexpr (kBytes % 16 == 0) {
    uint4 c[kBytes / 16];
#pragma unroll
    for (int k = 0; k < kBytes / 16; ++k) c[k] = lds128(p + 16 * k);
    memcpy(out, c, kBytes);
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k) out[k] = row[k];
  }
}

template <class T, class S>
constexpr uint32_t scan_tile_bytes() {
  return uint32_t(kScanThreads) * scan_items<S>() * uint32_t(sizeof(T));
}

template <class T, class S>
constexpr bool scan_tma_eligible() {
  return scan_tile_bytes<T, S>() % 16 == 0;
}

constexpr int kScanProducerThreads = 32;  // one producer warp (lane 0 works)
constexpr int kScanTmaThreads = kScanThreads + kScanProducerThreads;

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanTmaThreads) scan_tma_kernel(const ScanArgs<T, S, F, Op> a) {
  using A = typename ScanMath<S, Op>::A;
  constexpr int IT = scan_items<S>();
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  constexpr uint32_t kBytes = scan_tile_bytes<T, S>();
  constexpr int NW = kScanThreads / kWarp;
  extern __shared__ __align__(128) unsigned char stage_mem[];
  __shared__ __align__(8) uint64_t full[kScanStages];   // TMA landed (count 1 + tx)
  __shared__ __align__(8) uint64_t empty[kScanStages];  // consumers done (count NW)
  __shared__ uint32_t ring[kScanStages];
  __shared__ uint32_t s_epoch;
  __shared__ ScanSharedOf<S, Op> sh;

  const bool tail_partial = (a.n % kTile) != 0;
  if (threadIdx.x == kScanThreads) {
    for (int s = 0; s < kScanStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x >= kScanThreads) {
    // ---- producer warp: claims tiles in ticket order and keeps kScanStages
    // of them in flight.  The epoch is read BEFORE the first (acq_rel) claim;
    // each CTA claims until its first failure, so a launch makes exactly
    // ntiles + gridDim.x claims, and the last claimer resets the ticket and
    // advances the epoch for the next launch.
    if (threadIdx.x != kScanThreads) return;
    const uint32_t epoch = ld_acquire_gpu(a.ctrl + 2);
    s_epoch = epoch;
    for (uint32_t it = 0;; ++it) {
      const int s = int(it % kScanStages);
      if (it >= uint32_t(kScanStages)) mbar_wait(&empty[s], ((it / kScanStages) - 1) & 1u);
      uint32_t t = atom_add_acq_rel_gpu(a.ctrl + 0, 1u);
      if (t == a.ntiles + gridDim.x - 1) {
        st_relaxed_gpu(a.ctrl + 0, 0u);
        st_relaxed_gpu(a.ctrl + 2, epoch + 1u);
      }
      if (t >= a.ntiles) t = kNoTile;
      ring[s] = t;
      if (t != kNoTile && !(tail_partial && t == a.ntiles - 1)) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[s], kBytes);
        tma_load_1d(stage_mem + size_t(s) * kBytes, a.src + uint64_t(t) * kTile, kBytes, &full[s]);
      } else {
        mbar_arrive(&full[s]);  // end marker, or partial last tile read from global
      }
      if (t == kNoTile) return;
    }
  }

  // ---- 8 consumer warps
  for (uint32_t it = 0;; ++it) {
    const int s = int(it % kScanStages);
    mbar_wait(&full[s], (it / kScanStages) & 1u);
    const uint32_t tile = ring[s];
    if (tile == kNoTile) break;
    const uint32_t epoch = s_epoch;
    T raw[IT];
    int count;
    const uint64_t base = uint64_t(tile) * kTile + uint64_t(threadIdx.x) * IT;
    if (tail_partial && tile == a.ntiles - 1) {
      count = load_tile_items_global<T, IT>(a.src, 1, a.n, base, raw);
    } else {
      load_items_smem<T, IT>(reinterpret_cast<const T*>(stage_mem + size_t(s) * kBytes) + threadIdx.x * IT, raw);
      count = IT;
    }
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    scan_tile_body<T, S, F, Op, Inclusive, IT>(a, tile, epoch, raw, count, sh);
    consumer_sync();  // `sh` is reused by the next tile
  }
}

template <class T, class S, class Op>
struct ScanWs {
  using C = typename CarryTraits<S, Op>::C;
  static constexpr uint64_t kTile = uint64_t(kScanThreads) * scan_items<S>();
  static uint64_t tiles(uint64_t n) { return ceil_div(n, kTile); }
  // Each tile state owns a 256-byte slot (one L2-slice granule); larger
  // carries (> 256 B) take their natural size.
  static constexpr uint32_t kSlotWords =
      TileStateIO<C>::STRIDE > kStateSlotWords ? TileStateIO<C>::STRIDE : kStateSlotWords;
  static uint64_t bytes(uint64_t n) { return 256 + tiles(n) * kSlotWords * sizeof(uint64_t); }
};

template <class T, class S, class F, class Op, bool Inclusive>
inline uint32_t scan_tma_grid(uint64_t ntiles) {
  static thread_local int cached_dev = -1, cached_occ = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    const size_t smem = size_t(kScanStages) * scan_tile_bytes<T, S>();
    cudaFuncSetAttribute(scan_tma_kernel<T, S, F, Op, Inclusive>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scan_tma_kernel<T, S, F, Op, Inclusive>, kScanTmaThreads, smem);
    cached_occ = occ < 1 ? 1 : occ;
    cached_dev = dev;
  }
  const uint64_t cap = uint64_t(device_props().sm_count) * cached_occ;
  return uint32_t(ntiles < cap ? ntiles : cap);
}

// Kernel selection for contiguous aligned inputs: FORGE_SCAN_PATH=tma selects
// the persistent TMA kernel, anything else the one-tile-per-CTA kernel.
inline bool scan_use_tma() {
  static const bool v = [] {
    const char* e = std::getenv("FORGE_SCAN_PATH");
    return e && std::strcmp(e, "tma") == 0;
  }();
  return v;
}

// Experiment knobs (defaults are the tuned values): FORGE_SCAN_LOOKBACK = polls
// per thread of the block-wide look-back (0 = warp 0 only, window 32);
// FORGE_SCAN_STATE_WORDS = 64-bit words between consecutive tile states.
inline uint32_t scan_env_u32(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return e ? uint32_t(std::strtoul(e, nullptr, 10)) : dflt;
}
inline uint32_t scan_lookback_mode() {
  static const uint32_t v = scan_env_u32("FORGE_SCAN_LOOKBACK", 0);
  return v;
}
inline uint32_t scan_state_words_override() {
  static const uint32_t v = scan_env_u32("FORGE_SCAN_STATE_WORDS", 0);
  return v;
}

template <class T, class S, class F, class Op>
cudaError_t launch_scan(const T* src, uint64_t src_stride, S* dst, uint64_t dst_stride, uint64_t n,
                        bool inclusive, const F& f, const Op& op, const S& identity,
                        const S* carry_in, S* total_out, void* ws, cudaStream_t stream) {
  const uint64_t ntiles = ScanWs<T, S, Op>::tiles(n);
  if (ntiles == 0) return cudaSuccess;
  if (ntiles >= (1ull << 31)) return cudaErrorInvalidValue;
  ScanArgs<T, S, F, Op> a{src,      dst,       n,         src_stride, dst_stride,
                          f,        op,        identity,  carry_in,   total_out,
                          reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + 256),
                          static_cast<uint32_t*>(ws), uint32_t(ntiles),
                          ScanWs<T, S, Op>::kSlotWords, scan_lookback_mode()};
  {
    const uint32_t w = scan_state_words_override();
    if (w >= TileStateIO<typename CarryTraits<S, Op>::C>::STRIDE && w <= a.state_stride) a.state_stride = w;
  }
  const bool tma = scan_use_tma() && scan_tma_eligible<T, S>() && src_stride == 1 &&
                   is_aligned(src, 16) && ntiles >= 2;
  if (tma) {
    const size_t smem = size_t(kScanStages) * scan_tile_bytes<T, S>();
    if (inclusive)
      scan_tma_kernel<T, S, F, Op, true>
          <<<scan_tma_grid<T, S, F, Op, true>(ntiles), kScanTmaThreads, smem, stream>>>(a);
    else
      scan_tma_kernel<T, S, F, Op, false>
          <<<scan_tma_grid<T, S, F, Op, false>(ntiles), kScanTmaThreads, smem, stream>>>(a);
  } else {
    if (inclusive)
      scan_kernel<T, S, F, Op, true><<<uint32_t(ntiles), kScanThreads, 0, stream>>>(a);
    else
      scan_kernel<T, S, F, Op, false><<<uint32_t(ntiles), kScanThreads, 0, stream>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace forge::cuda
