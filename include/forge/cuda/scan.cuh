// forge/cuda/scan.cuh — single-pass decoupled look-back scan for sm_100a.
//
// Reference: prim::scan (primitives.hpp:440-603).  Same protocol (tile
// aggregate published as PARTIAL, look-back over predecessors until a PREFIX,
// own PREFIX published, outputs composed and stored once), re-designed for the
// hardware:
//   * tile ids: the TMA tile kernel uses blockIdx.x (its load starts at CTA
//     start; forward progress rests on in-order CTA dispatch, as in CUB's
//     single-pass scan — the VM admitted blocks in id order too,
//     machine.cpp:767-776); the lagged and register kernels take an atomic
//     ticket (deadlock-free under any dispatch order; scan_block_order);
//   * tile status: every 32-bit chunk of the published value travels in its
//     own 64-bit word {status, chunk}; a reader accepts a state only when all
//     words carry the same status — no fence, no separate flag byte (the
//     reference: relaxed aggregate store + release flag, primitives.hpp:518-534);
//   * each tile state owns a 256-byte slot: L2 slices are selected at 256-byte
//     granularity and every CTA in flight polls the newest tiles' states, so
//     packed 8-16-byte states put the hottest lines on ONE slice (measured
//     +25% scan bandwidth, profiles/);
//   * status = (epoch << 2) | {1 PARTIAL, 2 PREFIX}: every CTA gets the epoch
//     from its relaxed 64-bit {epoch, ticket} claim, and the LAST claimer
//     advances it for the next launch, so stale states of earlier launches
//     read as INVALID and the workspace needs no fill_zero per launch
//     (primitives.hpp:464-466);
//   * look-back: warp 0 polls 32 predecessors per L2 round trip, finds the
//     nearest PREFIX with one ballot and folds the window with a log-step
//     ORDER-PRESERVING reduction (the reference folded it serially,
//     primitives.hpp:561-563);
//   * cross-tile carries run in CarryTraits<S,Op>::C (f64 for the f32 sums);
//     product-type ops run entirely in C (ScanMath, reduce.cuh);
//   * optional carry_in (exclusive prefix of earlier shards) and total_out.
//
// Two kernels:
//   scan_smem_kernel  contiguous 16-byte-aligned inputs (the fast path): each
//                     CTA claims one tile of 256 rows x 128 bytes (8192 f32) and
//                     fetches it with ONE 2-D TMA (cp.async.bulk.tensor, 128-byte
//                     swizzle) into shared memory.  The tile is scanned in two
//                     passes over shared memory — pass 1 folds each thread's row
//                     to a total (-> block scan, look-back), pass 2 re-reads the
//                     row and emits running prefixes — so no item arrays live in
//                     registers: ~6 CTAs x 32 KB of HBM reads are in flight per
//                     SM, which Little's law needs at B200 latencies (the
//                     register-staged kernel tops out near 3.3 TB/s).
//   scan_kernel       everything else (strided views, unaligned bases): one
//                     tile of 256 x 64 bytes of S per CTA, direct vector /
//                     scalar loads into registers.
#pragma once

#include "forge/cuda/reduce.cuh"
#include "forge/cuda/tma.cuh"

namespace forge::cuda {

constexpr int kScanThreads = 256;
constexpr uint32_t kPartial = 1, kPrefix = 2;
constexpr uint32_t kStateSlotWords = 32;  // 256-byte tile-state slots
constexpr int kRowBytes = 128;            // smem kernel: bytes of T per thread row
constexpr uint32_t kLookbackSkipProbe = 99;  // FORGE_DEV builds only: FORGE_SCAN_LOOKBACK=99 skips the look-back
                                             // (WRONG results; the look-back-free ceiling probe of DESIGN.md §7)

constexpr int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Tile-state words.  Every 32-bit chunk of a published carry travels in its
// own 64-bit word {tag, chunk}, tag = (epoch << 2) | kind; a state is accepted
// only when all its words carry the same tag.  States are grouped P to a
// 32-byte sector (P = 4 / 2 / 1 for 1 / 2 / 4-word states) and the groups sit
// one per `stride`-word slot (256 bytes at full speed): one 256-bit load by a
// look-back lane reads P consecutive tiles, so a warp's poll round covers 32 * P
// predecessors for the same 32 L2 sector requests.
template <class C>
struct TileStateIO {
  static constexpr int SW = Words<C>::N;        // 32-bit chunks of the carry
  static constexpr int STRIDE = next_pow2(SW);  // 64-bit words per state: every chunk, any sizeof(C)
  static constexpr int P = STRIDE <= 4 ? 4 / STRIDE : 1;  // tiles per 32-byte group
  static constexpr int GW = STRIDE * P;                   // 64-bit words per group (>= 4)

  static __device__ __forceinline__ uint64_t* at(uint64_t* states, uint64_t tile, uint32_t stride) {
    return states + (tile / P) * stride + (tile % P) * STRIDE;
  }
  static __host__ __device__ constexpr uint64_t slots(uint64_t tiles) { return (tiles + P - 1) / P; }

  static __device__ __forceinline__ void write(uint64_t* states, uint64_t tile, uint32_t stride,
                                               uint32_t epoch, uint32_t kind, const C& v) {
    Words<C> w = to_words(v);
    const uint64_t hi = uint64_t((epoch << 2) | kind) << 32;
    uint64_t* p = at(states, tile, stride);
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

  // The whole group of slot `slot` (P tile states), 256-bit loads.
  static __device__ __forceinline__ void load_group(const uint64_t* states, uint64_t slot, uint32_t stride,
                                                    uint64_t (&raw)[GW]) {
    const uint64_t* p = states + slot * stride;
#pragma unroll
    for (int i = 0; i < GW; i += 4) ld_relaxed_gpu_v4(p + i, raw[i], raw[i + 1], raw[i + 2], raw[i + 3]);
  }
  // The state's kind from its tags alone (value not decoded); 0 = INVALID.
  static __device__ __forceinline__ uint32_t kind_of(const uint64_t* raw, uint32_t epoch) {
    const uint32_t hi = uint32_t(raw[0] >> 32);
    bool same = true;
#pragma unroll
    for (int i = 1; i < SW; ++i) same &= uint32_t(raw[i] >> 32) == hi;
    return same && (hi >> 2) == (epoch & 0x3fffffffu) ? hi & 3u : 0u;
  }
  // Decodes the state at word offset `off` of a group; 0 = INVALID.
  static __device__ __forceinline__ uint32_t decode(const uint64_t* raw, uint32_t epoch, C& v,
                                                   uint32_t epoch_mask = 0x3fffffffu) {
    const uint32_t hi = uint32_t(raw[0] >> 32);
    bool same = true;
#pragma unroll
    for (int i = 1; i < SW; ++i) same &= uint32_t(raw[i] >> 32) == hi;
    const uint32_t kind = hi & 3u;
    if (!same || kind == 0 || ((hi >> 2) & epoch_mask) != (epoch & epoch_mask)) return 0;
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
  uint64_t* states;   // tile states, state_stride words apart
  uint32_t* ctrl;     // 64-bit control word: {epoch (high 32), ticket (low 32)}
  uint32_t ntiles;
  uint32_t state_stride;  // 64-bit words per tile state slot
  uint32_t lookback;      // 0 (FORGE_DEV builds: kLookbackSkipProbe skips the look-back)
  uint64_t* trace;        // FORGE_DEV builds: per-tile phase timestamps (own buffer), else null
  uint32_t backoff_ns;    // look-back: sleep between polls of INVALID states (0; FORGE_DEV knob)
  uint32_t epoch_mask;    // 0x3fffffff; 0 = the relax_scan_flag ablation (MutationFlags,
                          // primitives.hpp:64-67): stale states of earlier launches are accepted
  uint64_t perturb_seed;  // test schedule perturbation (ScanTestHooks), 0 = off
  uint32_t perturb_ns;
  uint32_t prefetch_ahead;  // CTA g L2-prefetches tile g + prefetch_ahead (0: tile g; scan_prefetch_ahead)
  uint32_t block_order;     // scan_smem_kernel: tile = blockIdx.x, loaded at CTA start (scan_block_order)
};

// Test-only hooks of one scan launch (both off in production):
//   relax_epoch   the relax_scan_flag ablation (MutationFlags, reference
//                 primitives.hpp:64-67): the epoch tag of tile states is
//                 ignored, so a state left by an earlier launch on the same
//                 workspace is accepted as if it were published by this one;
//   perturb_seed  the B200 counterpart of the simulator's adversarial
//   perturb_ns    schedules (ScheduleSeed, machine.hpp): a pseudo-random 1/8 of
//                 the tiles (chosen by the seed) wait perturb_ns before
//                 publishing their aggregate, so successors poll states that
//                 are not yet published.  Measured on B200: without it no tile
//                 ever polls an unpublished predecessor (CTAs launch, load and
//                 publish in ticket order), and the ablation goes unseen.
struct ScanTestHooks {
  bool relax_epoch = false;
  uint64_t perturb_seed = 0;
  uint32_t perturb_ns = 0;
};

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase timestamps of a tile: 0 claimed, 1 data landed, 2 pass 1 done,
// 3 prefix known (look-back done), 4 pass 2 done; 5 = SM id, 6 = look-back
// rounds, 7 = CTA start (before the speculative TMA and the claim).
__device__ __forceinline__ void trace_mark(uint64_t* trace, uint64_t tile, int phase) {
  if (trace && threadIdx.x == 0) trace[tile * 8 + phase] = global_ns();
}

constexpr int kMaxSubtiles = 2;  // 32 KB sub-tiles per CTA tile (smem kernel, scan_subtiles)

template <class A, class C>
struct ScanShared {
  Opt<A> warp[kMaxSubtiles * kScanThreads / kWarp];
  Opt<A> carry;
};

template <class S, class Op>
using ScanSharedOf = ScanShared<typename ScanMath<S, Op>::A, typename ScanMath<S, Op>::C>;

// Decoupled look-back by one warp (primitives.hpp:536-576).  Each round, lane
// l reads state group (top - l) with one 256-bit load — P consecutive tiles —
// re-polls only while its group holds an INVALID state newer than its newest
// PREFIX, and pre-folds its group newest-to-oldest (stopping at a PREFIX).
// One ballot then finds the nearest lane holding a PREFIX and the lanes newer
// than it are folded with an ORDER-PRESERVING log-step reduction (older
// always on the left; the reference folded serially, :561-563).  Returns the
// carry (all lanes).
// Measured (tools/trace_scan.py, f32 2^28, one tile per lane): the nearest
// PREFIX sits ~100 tiles back under load and a poll round costs 1.7-3 us
// (tools/probe_rtt.cu: L2-hit latency under full HBM streaming), so the
// window per round, not the number of loads, sets the look-back time.
template <class IO, class C, class COp>
__device__ __forceinline__ Opt<C> warp_lookback(const uint64_t* states, uint32_t stride, uint32_t epoch,
                                                int64_t tile, const COp& cop, uint64_t* trace, uint64_t trace_tile,
                                                uint32_t backoff_ns, uint32_t epoch_mask) {
  constexpr uint32_t kEmpty = 4;  // group before tile 0
  constexpr int P = IO::P;
  const unsigned lane = lane_id();
  Opt<C> carry{C{}, false};
  int64_t top = (tile - 1) / P;  // group of the newest predecessor
  uint32_t rounds = 0;
  for (;;) {
    ++rounds;
    const int64_t slot = top - int64_t(lane);
    uint32_t kind = slot < 0 ? kEmpty : 0u;  // lane summary: PARTIAL / PREFIX / kEmpty; 0 = re-poll
    Opt<C> val{C{}, false};
    for (;;) {
      if (kind == 0) {
        uint64_t raw[IO::GW];
        IO::load_group(states, uint64_t(slot), stride, raw);
        Opt<C> acc{C{}, false};
        uint32_t k = kPartial;
#pragma unroll
        for (int q = P - 1; q >= 0; --q) {
          if (k != kPartial || slot * P + q >= tile) continue;  // resolved, or not a predecessor
          C v;
          const uint32_t kq = IO::decode(raw + q * IO::STRIDE, epoch, v, epoch_mask);
          if (kq == 0) {
            k = 0;
          } else {
            acc = opt_combine(cop, Opt<C>{v, true}, acc);
            if (kq == kPrefix) k = kPrefix;
          }
        }
        kind = k;
        val = acc;
      }
      if (__all_sync(kFullMask, kind != 0)) break;
      if (backoff_ns) __nanosleep(backoff_ns);
    }
    const unsigned pm = __ballot_sync(kFullMask, kind == kPrefix);
    const int near = pm ? __ffs(int(pm)) - 1 : kWarp;  // lane of the nearest PREFIX (kWarp: none)
    Opt<C> v{val.v, int(lane) <= near && kind != kEmpty && val.has};
#pragma unroll
    for (unsigned d = 1; d < kWarp; d <<= 1) {
      Opt<C> got{shfl_down(v.v, d), __shfl_down_sync(kFullMask, int(v.has), d) != 0};
      if (lane + d < kWarp) v = opt_combine(cop, got, v);
    }
    carry = opt_combine(cop, shfl_idx_opt(v, 0), carry);
    if (near < kWarp || top < kWarp) break;  // found a PREFIX, or reached tile 0
    top -= kWarp;
  }
  if (trace && lane == 0) trace[trace_tile * 8 + 6] = rounds;
  return carry;
}

// Claims the next tile: ONE 64-bit atomic on the control word {epoch:32,
// ticket:32} returns the ticket and this launch's epoch together (one L2
// round trip, ~2 us under full HBM load — a separate epoch load before the
// ticket would be a second, serial one).  The last of the `ntiles` claims
// resets the ticket and advances the epoch for the next launch; no CTA of this
// launch touches the word after it.
template <class T, class S, class F, class Op>
__device__ __forceinline__ uint32_t claim_tile(const ScanArgs<T, S, F, Op>& a, uint32_t& epoch) {
  uint64_t* word = reinterpret_cast<uint64_t*>(a.ctrl);
  const uint64_t got = atom_add_relaxed_gpu(word, uint64_t(1));  // see scan_lag_kernel's claim
  const uint32_t t = uint32_t(got);
  epoch = uint32_t(got >> 32);
  if (t == a.ntiles - 1) st_relaxed_gpu(word, uint64_t(epoch + 1u) << 32);
  return t;
}

// Block scan of the per-thread totals, publication of the tile aggregate, the
// decoupled look-back, publication of the tile's inclusive prefix.  Returns the
// EXCLUSIVE prefix of this thread (everything before its first item, carry and
// earlier tiles included); `.has == false` only for the very first item of a
// carry-less scan.
//
// R > 1: every thread holds R values — value r of thread t sits at position
// r * kScanThreads + t of the tile (sub-tile r); all R * #warps warp totals are
// scanned by warp 0 at once (R * 8 <= 32).
template <int R, class T, class S, class F, class Op>
__device__ __forceinline__ void block_exclusive_prefix(
    const ScanArgs<T, S, F, Op>& a, uint64_t tile, uint32_t epoch,
    const Opt<typename ScanMath<S, Op>::A> (&thread_total)[R], ScanSharedOf<S, Op>& sh,
    Opt<typename ScanMath<S, Op>::A> (&ex)[R]) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  constexpr int NW = kScanThreads / kWarp;
  static_assert(R >= 1 && R <= kMaxSubtiles && R * NW <= kWarp, "sub-tiles per CTA");
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };

  // ---- warp scans, cross-warp scan through shared memory (:501-516)
  Opt<A> incl[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    incl[r] = warp_scan_incl(aop, thread_total[r]);
    if (lane == kWarp - 1) sh.warp[r * NW + warp] = incl[r];
  }
  __syncthreads();
  if (warp == 0) {
    Opt<A> w = lane < R * NW ? sh.warp[lane] : Opt<A>{A{}, false};
    w = warp_scan_incl(aop, w);
    if (lane < R * NW) sh.warp[lane] = w;
  }
  __syncthreads();
  const Opt<A> agg = sh.warp[R * NW - 1];  // every tile holds >= 1 element

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
    const C agg_c = M::to_c(agg.v);
    if (threadIdx.x == 0) {
      if (a.perturb_ns && ((tile * 0x9E3779B97F4A7C15ull) ^ a.perturb_seed) % 8 == 0) {  // test hook
        const uint64_t t0 = global_ns();
        while (global_ns() - t0 < a.perturb_ns) __nanosleep(200);
      }
      IO::write(a.states, tile, a.state_stride, epoch, kPartial, agg_c);
    }
    Opt<C> carry{C{}, false};  // meaningful in thread 0
    if (a.lookback == kLookbackSkipProbe) {
      // development ceiling probe (FORGE_SCAN_LOOKBACK=99): no look-back, WRONG results
    } else if (warp == 0) {
      carry = warp_lookback<IO, C>(a.states, a.state_stride, epoch, int64_t(tile), cop, a.trace, tile, a.backoff_ns,
                                   a.epoch_mask);
    }
    if (threadIdx.x == 0) {
      const C inclusive_c = cop(carry.v, agg_c);
      IO::write(a.states, tile, a.state_stride, epoch, kPrefix, inclusive_c);
      sh.carry = Opt<A>{M::from_c(carry.v), true};
      if (tile == a.ntiles - 1 && a.total_out) *a.total_out = M::CT::to_s(inclusive_c);
    }
  }
  __syncthreads();

  const Opt<A> tile_ex = sh.carry;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int wi = r * NW + int(warp);
    const Opt<A> warp_ex = wi > 0 ? sh.warp[wi - 1] : Opt<A>{A{}, false};
    Opt<A> lane_ex = shfl_up_opt(incl[r], 1);
    if (lane == 0) lane_ex.has = false;
    ex[r] = opt_combine(aop, opt_combine(aop, tile_ex, warp_ex), lane_ex);
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
// General path: one register-staged tile per CTA.

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const ScanArgs<T, S, F, Op> a) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  constexpr int IT = scan_items<S>();
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ ScanSharedOf<S, Op> sh;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  if (threadIdx.x == 0) {
    uint32_t e;
    s_tile = claim_tile(a, e);
    s_epoch = e;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * IT;
  T raw[IT];
  const int count = load_tile_items_global<T, IT>(a.src, a.src_stride, a.n, base, raw);

  // per-thread register scan (primitives.hpp:484-499)
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

  const Opt<A> tot1[1] = {Opt<A>{last, count > 0}};
  Opt<A> pre1[1];
  block_exclusive_prefix<1>(a, tile, s_epoch, tot1, sh, pre1);
  const Opt<A> pre = pre1[0];
  if (count == 0) return;

  // compose outputs in registers and store once (:579-600)
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

// ---------------------------------------------------------------------------
// Fast path: TMA-loaded shared-memory tile, two passes.

template <class T>
constexpr bool smem_scan_type_ok() {
  return sizeof(T) == 1 || sizeof(T) == 2 || sizeof(T) == 4 || sizeof(T) == 8 || sizeof(T) == 16;
}

template <class T>
constexpr int smem_scan_items() {
  return kRowBytes / int(sizeof(T)) > 0 ? kRowBytes / int(sizeof(T)) : 1;
}

constexpr uint32_t kSmemTileBytes = uint32_t(kScanThreads) * kRowBytes;  // 32 KB
constexpr uint32_t kSmemScanDyn = kSmemTileBytes + 1024;                 // + swizzle alignment slack

// `tmap_out` (used when tma_store) views dst as 128-byte rows; only for
// sizeof(S) == sizeof(T), where each output chunk overwrites its input chunk
// in shared memory and the finished tile leaves with one TMA tensor store.
//
// R sub-tiles per CTA: the tile is R x 32 KB (R boxes of 256 rows); thread t
// owns row t of every sub-tile.  R = 2 halves the number of tile states, of
// look-back pollers and of the claim rate for the same bytes in flight (the
// look-back's lag and its per-round latency both scale with them).
//
// Resident CTAs per SM the kernel is compiled for: 6 x 33 KB (R = 1) or
// 3 x 65 KB (R = 2) of tile (Little's law) — <= 40 / 80
// registers.
// Wide carries (f64 affine / quaternion, 16-byte structs) get the same 6
// CTAs/SM: measured affine 2^28 at 4 / 5 / 6 CTAs/SM (64 / 48 / 40 registers,
// the last with 20 bytes of spills): 3,744 / 4,193 / 4,252 GB/s.
#ifndef FORGE_SCAN_WIDE_BLOCKS
#define FORGE_SCAN_WIDE_BLOCKS 6
#endif
constexpr int scan_env_wide_blocks() { return FORGE_SCAN_WIDE_BLOCKS; }

template <class S, class Op, int R>
constexpr int scan_smem_min_blocks() {
  return (sizeof(typename ScanMath<S, Op>::C) <= 8 ? 6 : scan_env_wide_blocks()) / R;
}

constexpr uint32_t scan_smem_dyn(int R) { return uint32_t(R) * kSmemTileBytes + 1024; }

template <class T, class S, class F, class Op, bool Inclusive, int R>
__global__ void __launch_bounds__(kScanThreads, scan_smem_min_blocks<S, Op, R>())
    scan_smem_kernel(const ScanArgs<T, S, F, Op> a, const __grid_constant__ CUtensorMap tmap,
                     const __grid_constant__ CUtensorMap tmap_out, bool tma_store) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  constexpr int IT = smem_scan_items<T>();  // items per thread row (one 128-byte row)
  constexpr int EPC = 16 / int(sizeof(T));  // items per 16-byte chunk
  constexpr int NCH = kRowBytes / 16;       // chunks per row
  constexpr uint64_t kSub = uint64_t(kScanThreads) * IT;  // items per sub-tile
  constexpr uint64_t kTile = kSub * R;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tile, s_epoch, s_phase;
  __shared__ ScanSharedOf<S, Op> sh;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  unsigned char* tile_mem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  auto load_tile = [&](uint32_t t) {
    mbar_arrive_expect_tx(&bar, uint32_t(R) * kSmemTileBytes);
#pragma unroll
    for (int r = 0; r < R; ++r)
      tma_load_2d(tile_mem + size_t(r) * kSmemTileBytes, &tmap, 0, (int(t) * R + r) * kScanThreads, &bar);
  };

  const uint64_t t_start = a.trace ? global_ns() : 0;
  if (threadIdx.x == 0) {
    // Tile blockIdx.x is prefetched into L2 BEFORE the ticket round trip; the
    // ticket stays the source of truth, and the tile it names was prefetched
    // by the CTA of that index, which started at about the same time (tickets
    // match blockIdx.x for only 1-3 % of CTAs, but are close to it), so the
    // shared-memory load after the claim is an L2 hit.  (A speculative
    // shared-memory load of blockIdx.x had to land before the claimed tile
    // could be loaded: 2^28 lagged f32 5.60 -> 5.88 TB/s with the prefetch.)
    const uint32_t g = blockIdx.x;
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint64_t gp = uint64_t(g) + a.prefetch_ahead;
    auto prefetch = [&](uint64_t t) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        tma_prefetch_2d_hint(&tmap, 0, (int(t) * R + r) * kScanThreads, l2_policy_evict_normal());
    };
    if (a.block_order) {
      // Tile g itself: its HBM load starts at once and the claim (kept for
      // the launch epoch and the ticket reset) overlaps it.
      if (uint64_t(g + 1) * kTile <= a.n) load_tile(g);
      if ((gp + 1) * kTile <= a.n) prefetch(gp);
      uint32_t e;
      claim_tile(a, e);
      s_tile = g;
      s_epoch = e;
      s_phase = 0;
    } else {
      if (a.prefetch_ahead && g < a.prefetch_ahead && uint64_t(g + 1) * kTile <= a.n) prefetch(g);
      if ((gp + 1) * kTile <= a.n) prefetch(gp);
      uint32_t e;
      const uint32_t t = claim_tile(a, e);
      s_tile = t;
      s_epoch = e;
      s_phase = 0;
      if (uint64_t(t + 1) * kTile <= a.n) load_tile(t);
    }
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  trace_mark(a.trace, tile, 0);
  if (a.trace && threadIdx.x == 0) {
    uint32_t sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    a.trace[tile * 8 + 5] = sm;
    a.trace[tile * 8 + 7] = t_start;
  }
  const bool full = (tile + 1) * kTile <= a.n;
  uint64_t base[R];
  int count[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    base[r] = tile * kTile + uint64_t(r) * kSub + uint64_t(threadIdx.x) * IT;
    const uint64_t avail = base[r] < a.n ? a.n - base[r] : 0;
    count[r] = full ? IT : (avail >= uint64_t(IT) ? IT : int(avail));
  }

  // ---- pass 1: ordered fold of this thread's rows
  Opt<A> tot[R];
  if (full) {
    mbar_wait(&bar, s_phase);
    trace_mark(a.trace, tile, 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const unsigned char* tm = tile_mem + size_t(r) * kSmemTileBytes;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint4 v = lds128(tm + swz128(threadIdx.x, c));
        T x[EPC];
        memcpy(x, &v, 16);
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const A y = M::lift(a.f(x[e]));
          tot[r].v = (c == 0 && e == 0) ? y : aop(tot[r].v, y);
        }
      }
      tot[r].has = true;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      tot[r] = Opt<A>{A{}, false};
      for (int k = 0; k < count[r]; ++k) {
        const A y = M::lift(a.f(a.src[base[r] + k]));
        tot[r].v = k == 0 ? y : aop(tot[r].v, y);
      }
      tot[r].has = count[r] > 0;
    }
  }

  trace_mark(a.trace, tile, 2);
  Opt<A> run[R];
  block_exclusive_prefix<R>(a, tile, s_epoch, tot, sh, run);
  trace_mark(a.trace, tile, 3);

  // ---- pass 2: running prefixes, stored as they are produced.  E is the
  // type of the running value: A, or S for kNarrowEmit ops (the f64 exclusive
  // prefix rounded once, then the row's items composed in S).
  using E = std::conditional_t<M::kNarrowEmit, S, A>;
  Opt<E> emit[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if constexpr (M::kNarrowEmit)
      emit[r] = Opt<E>{M::lower(run[r].v), run[r].has};
    else
      emit[r] = run[r];
  }
  auto eop = [&](const E& x, const E& y) {
    if constexpr (M::kNarrowEmit)
      return a.op(x, y);
    else
      return aop(x, y);
  };
  auto elift = [&](const S& y) {
    if constexpr (M::kNarrowEmit)
      return y;
    else
      return M::lift(y);
  };
  auto elower = [&](const E& v) {
    if constexpr (M::kNarrowEmit)
      return v;
    else
      return M::lower(v);
  };
  if (full) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unsigned char* tm = tile_mem + size_t(r) * kSmemTileBytes;
      const bool vec = is_aligned(a.dst + base[r], 16);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint4 v = lds128(tm + swz128(threadIdx.x, c));
        T x[EPC];
        memcpy(x, &v, 16);
        S o[EPC];
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const E y = elift(a.f(x[e]));
          if constexpr (Inclusive) {
            emit[r].v = emit[r].has ? eop(emit[r].v, y) : y;
            emit[r].has = true;
            o[e] = elower(emit[r].v);
          } else {
            o[e] = emit[r].has ? elower(emit[r].v) : a.identity;
            emit[r].v = emit[r].has ? eop(emit[r].v, y) : y;
            emit[r].has = true;
          }
        }
        if constexpr (sizeof(S) == sizeof(T)) {
          if (tma_store) {
            uint4 w;
            memcpy(&w, o, 16);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(tm + swz128(threadIdx.x, c))),
                         "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                         : "memory");
            continue;
          }
        }
        S* d = a.dst + base[r] + uint64_t(c) * EPC;
        if (vec) {
          store_items<S, EPC>(d, o);
        } else {
#pragma unroll
          for (int e = 0; e < EPC; ++e) d[e] = o[e];
        }
      }
    }
    if (sizeof(S) == sizeof(T) && tma_store) {
      fence_proxy_async_smem();  // generic smem writes -> visible to the TMA engine
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          tma_store_2d(&tmap_out, 0, (int(tile) * R + r) * kScanThreads, tile_mem + size_t(r) * kSmemTileBytes);
        tma_store_commit();
        tma_store_wait_read();  // keep the CTA (and its smem) alive until read
      }
    }
    trace_mark(a.trace, tile, 4);
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      for (int k = 0; k < count[r]; ++k) {
        const E y = elift(a.f(a.src[base[r] + k]));
        if constexpr (Inclusive) {
          emit[r].v = emit[r].has ? eop(emit[r].v, y) : y;
          emit[r].has = true;
          a.dst[base[r] + k] = elower(emit[r].v);
        } else {
          a.dst[base[r] + k] = emit[r].has ? elower(emit[r].v) : a.identity;
          emit[r].v = emit[r].has ? eop(emit[r].v, y) : y;
          emit[r].has = true;
        }
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Lagged scan: the look-back moved off the tile's critical path.
//
// Ticket k does two things with ONE 32 KB shared-memory tile buffer:
//   A(k)      TMA-load tile k from HBM (L2 evict_last: it is read again soon),
//             fold it to its aggregate, publish the aggregate (tile state,
//             written once).  The A of the last tile of a 32-tile GROUP also
//             folds the group's 32 aggregates and publishes the group
//             aggregate (group state kind PARTIAL).
//   B(k - D)  the scan of tile j = k - D, D tiles behind: re-load it (an L2 hit:
//             D tiles of reads + writes stay well inside the 126 MB L2), fold
//             its rows, compose with the tile's exclusive prefix, emit, TMA
//             store; the last tile of a group publishes the group's inclusive
//             prefix (group state kind PREFIX).
// j's exclusive prefix needs only states published by LOWER tickets' A phases
// (tile aggregates of j's group, group aggregates) plus, as a shortcut, group
// PREFIXes of finished B phases: warp 0 reads them — one 32-lane round of
// tile aggregates and one of group states, issued together — WHILE A's HBM
// load is in flight, so the look-back round trips (2-3 us under load,
// tools/probe_rtt.cu) overlap the load instead of extending the tile's life.
// Every wait is on a lower ticket's A phase, which waits on nothing but lower
// tickets: deadlock-free under ticket order like the single-pass kernel.
//
// Full tiles only; a partial last tile is scanned by a second (tail) launch
// seeded with the full tiles' total.
constexpr uint32_t kLagGroup = 32;  // tiles per group

template <class T, class S, class F, class Op>
struct LagArgs {
  ScanArgs<T, S, F, Op> s;  // src, dst, f, op, identity, carry_in, total_out, ctrl, ntiles (full tiles)
  uint64_t* tagg;           // tile aggregates: STRIDE words per tile, compact
  uint64_t* gstate;         // group states: STRIDE words per group, compact
  uint32_t lag;             // D
  uint32_t nclaims;         // ntiles + D
};

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads, 6)
    scan_lag_kernel(const LagArgs<T, S, F, Op> L, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ CUtensorMap tmap_out) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  constexpr int ST = IO::STRIDE;
  constexpr int IT = smem_scan_items<T>();
  constexpr int EPC = 16 / int(sizeof(T));
  constexpr int NCH = kRowBytes / 16;
  constexpr int NW = kScanThreads / kWarp;
  const auto& a = L.s;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_k, s_epoch;
  __shared__ Opt<A> s_warp[NW];
  __shared__ Opt<C> s_carry;
  __shared__ C s_carry_agg;  // A's tile aggregate
  __shared__ C s_self_agg;   // B's tile aggregate (published by A(j))
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };
  unsigned char* buf =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  uint64_t* const tr = a.trace;  // FORGE_DEV builds: per-ticket phase stamps (tools/trace_lag.py)
  const uint64_t t_start = tr ? global_ns() : 0;

  // ---- claim.  Tile blockIdx.x is fetched into L2 while the claim is in
  // flight: tickets follow CTA start order only roughly (97-99 % of CTAs get a
  // ticket other than blockIdx.x, tools/trace_lag.py), but the tile a CTA
  // claims was prefetched by the CTA with that index, which started at about
  // the same time, so its shared-memory load right after the claim is an L2
  // hit (or joins the fill in flight).  A speculative shared-memory load of
  // blockIdx.x instead had to land before the buffer could take the claimed
  // tile (affine 5.24 -> 5.62 TB/s with the prefetch).
  if (threadIdx.x == 0) {
    const uint32_t g = blockIdx.x;
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint64_t pol = l2_policy_evict_last();
    if (a.block_order) {  // ticket = blockIdx.x (scan_block_order): A's load starts before the claim
      if (g < a.ntiles) {
        mbar_arrive_expect_tx(&bar, kSmemTileBytes);
        tma_load_2d_hint(buf, &tmap, 0, int(g) * kScanThreads, &bar, pol);
      }
    } else if (g < a.ntiles) {
      tma_prefetch_2d_hint(&tmap, 0, int(g) * kScanThreads, pol);
    }
    uint64_t* word = reinterpret_cast<uint64_t*>(a.ctrl);
    // relaxed: nothing is ordered by the claim (every tile state carries its
    // launch's epoch; the workspace memset precedes the launch).  An acq_rel
    // RMW costs a MEMBAR.ALL.GPU + ERRBAR before it and an L1 invalidate
    // after, measured 2^28 f32 5,290 -> 5,530 GB/s, affine 4,900 -> 5,110,
    // Mat2 4,930 -> 5,100 without them.
    const uint64_t got = atom_add_relaxed_gpu(word, uint64_t(1));
    const uint32_t t = uint32_t(got);
    const uint32_t e = uint32_t(got >> 32);
    if (t == L.nclaims - 1) st_relaxed_gpu(word, uint64_t(e + 1u) << 32);
    const uint32_t k = a.block_order ? g : t;
    s_k = k;
    s_epoch = e;
    if (!a.block_order && k < a.ntiles) {
      mbar_arrive_expect_tx(&bar, kSmemTileBytes);
      tma_load_2d_hint(buf, &tmap, 0, int(k) * kScanThreads, &bar, pol);
    }
  }
  __syncthreads();
  const uint32_t k = s_k, epoch = s_epoch;
  uint32_t phase = 0;  // parity of the barrier's next completion
  if (tr && threadIdx.x == 0) {
    tr[uint64_t(k) * 8 + 0] = t_start;
    tr[uint64_t(k) * 8 + 1] = (global_ns() & ~uint64_t(1)) | uint64_t(k != blockIdx.x);  // LSB: ticket != blockIdx.x
  }
  const bool hasA = k < a.ntiles;
  const bool hasB = k >= L.lag && k - L.lag < a.ntiles;
  const uint64_t j = uint64_t(k) - L.lag;  // B's tile

  // ---- warp 0: B's exclusive prefix, while A's tile is in flight
  if (hasB && warp == 0) {
    const uint64_t grp = j / kLagGroup;
    const uint32_t r = uint32_t(j % kLagGroup);
    // B publishes the group PREFIX (last tile of a group) / the total (last
    // tile): it needs tile j's own aggregate too (lane r)
    const bool want_self = r == kLagGroup - 1 || j == a.ntiles - 1;
    Opt<C> carry{C{}, false};
    // in-group: aggregates of tiles grp*32 .. j-1 (lane l: tile grp*32 + l).
    // The group's state has two writers — A(j) of its last tile (PARTIAL) and
    // B of that tile (PREFIX, below) — so B waits until A's PARTIAL is in
    // (lane 0): a state wider than one 128-bit store could otherwise end up
    // torn between the two (a permanently invalid state: measured as a rare
    // hang with 16-byte carries), and a late PARTIAL would hide the PREFIX.
    Opt<C> ing{C{}, false};
    {
      C v{};
      bool ok = !(lane < r || (lane == r && want_self));
      while (true) {
        if (!ok) {
          uint64_t raw[ST];
          const uint64_t* p = L.tagg + (grp * kLagGroup + lane) * ST;
#pragma unroll
          for (int i = 0; i < ST; i += 2) {
            if constexpr (ST == 1) raw[0] = ld_relaxed_gpu(p);
            else ld_relaxed_gpu_v2(p + i, raw[i], raw[i + 1]);
          }
          ok = IO::decode(raw, epoch, v, a.epoch_mask) != 0;
        }
        if (__all_sync(kFullMask, ok)) break;
      }
      if (r == kLagGroup - 1 && lane == 0) {  // (usually in long before: A(j) ran D tickets ago)
        while (true) {
          uint64_t raw[ST];
          const uint64_t* p = L.gstate + grp * ST;
#pragma unroll
          for (int i = 0; i < ST; i += 2) {
            if constexpr (ST == 1) raw[0] = ld_relaxed_gpu(p);
            else ld_relaxed_gpu_v2(p + i, raw[i], raw[i + 1]);
          }
          if (IO::kind_of(raw, epoch) == kPartial) break;  // this launch's (never the relaxed-epoch test mask)
        }
      }
      __syncwarp();
      if (want_self && lane == r) s_self_agg = v;
      Opt<C> x{v, lane < r};
      // ordered fold of lanes 0..r-1 (lane order = tile order)
#pragma unroll
      for (unsigned d = 1; d < kWarp; d <<= 1) {
        Opt<C> got{shfl_down(x.v, d), __shfl_down_sync(kFullMask, int(x.has), d) != 0};
        if (lane + d < kWarp) x = opt_combine(cop, x, got);
      }
      ing = shfl_idx_opt(x, 0);
    }
    // group level: states of groups grp-1, grp-2, ... (lane l: group top - l)
    int64_t top = int64_t(grp) - 1;
    Opt<C> grp_carry{C{}, false};
    bool reached_start = top < 0;
    while (top >= 0) {
      const int64_t gi = top - int64_t(lane);
      uint32_t kind = gi < 0 ? 4u : 0u;
      C v{};
      while (true) {
        if (kind == 0) {
          uint64_t raw[ST];
          const uint64_t* p = L.gstate + uint64_t(gi) * ST;
#pragma unroll
          for (int i = 0; i < ST; i += 2) {
            if constexpr (ST == 1) raw[0] = ld_relaxed_gpu(p);
            else ld_relaxed_gpu_v2(p + i, raw[i], raw[i + 1]);
          }
          kind = IO::decode(raw, epoch, v, a.epoch_mask);
        }
        if (__all_sync(kFullMask, kind != 0)) break;
      }
      const unsigned pm = __ballot_sync(kFullMask, kind == kPrefix);
      const int near = pm ? __ffs(int(pm)) - 1 : kWarp;
      Opt<C> x{v, int(lane) <= near && kind != 4u};
#pragma unroll
      for (unsigned d = 1; d < kWarp; d <<= 1) {  // older (higher lane) on the left
        Opt<C> got{shfl_down(x.v, d), __shfl_down_sync(kFullMask, int(x.has), d) != 0};
        if (lane + d < kWarp) x = opt_combine(cop, got, x);
      }
      grp_carry = opt_combine(cop, shfl_idx_opt(x, 0), grp_carry);
      if (near < kWarp) break;
      if (top < int64_t(kWarp)) {
        reached_start = true;
        break;
      }
      top -= kWarp;
    }
    if (reached_start && a.carry_in) carry = Opt<C>{M::CT::to_c(*a.carry_in), true};
    carry = opt_combine(cop, carry, grp_carry);
    carry = opt_combine(cop, carry, ing);
    if (lane == 0) s_carry = carry;
    if (tr && lane == 0) tr[uint64_t(k) * 8 + 4] = global_ns();
  }

  // The tile in `buf` folded and block-scanned (A: its aggregate, passed to
  // on_aggregate by warp 0 lane NW-1; B: also this row's exclusive prefix
  // inside the tile, (warps before) o (lanes before)).  A and B run the same
  // tree, so A's published aggregate and B's PREFIX are the same bits.
  auto tile_row_prefix = [&](auto want_row, auto sync_first, auto&& on_aggregate) -> Opt<A> {
    Opt<A> tot;
    auto fold_chunk = [&](int c) {
      const uint4 v = lds128(buf + swz128(threadIdx.x, c));
      T x[EPC];
      memcpy(x, &v, 16);
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const A y = M::lift(a.f(x[e]));
        tot.v = (c == 0 && e == 0) ? y : aop(tot.v, y);
      }
    };
    if constexpr (sizeof(A) >= 16) {  // wide accumulators: fewer row chunks in flight (no spill at 40 registers)
#pragma unroll 2
      for (int c = 0; c < NCH; ++c) fold_chunk(c);
    } else {
#pragma unroll
      for (int c = 0; c < NCH; ++c) fold_chunk(c);
    }
    tot.has = true;
    const Opt<A> incl = warp_scan_incl(aop, tot);
    if constexpr (decltype(sync_first)::value) __syncthreads();  // s_warp: earlier readers are done
    if (lane == kWarp - 1) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      Opt<A> w = lane < NW ? s_warp[lane] : Opt<A>{A{}, false};
      w = warp_scan_incl(aop, w);
      if constexpr (decltype(want_row)::value) {
        if (lane < NW) s_warp[lane] = w;
      }
      if (lane == NW - 1) on_aggregate(w.v);  // the tile aggregate
    }
    __syncthreads();
    if constexpr (decltype(want_row)::value) {
      const Opt<A> warp_ex = warp > 0 ? s_warp[warp - 1] : Opt<A>{A{}, false};
      Opt<A> lane_ex = shfl_up_opt(incl, 1);
      if (lane == 0) lane_ex.has = false;
      return opt_combine(aop, warp_ex, lane_ex);
    } else {
      return Opt<A>{A{}, false};
    }
  };

  // ---- A: fold tile k, publish its aggregate
  if (hasA) {
    mbar_wait(&bar, phase);
    phase ^= 1u;
    if (tr && threadIdx.x == 0) tr[uint64_t(k) * 8 + 2] = global_ns();
    tile_row_prefix(std::false_type{}, std::false_type{}, [&](const A& total) {
          const C agg = M::to_c(total);
          s_carry_agg = agg;
          if (a.perturb_ns && ((uint64_t(k) * 0x9E3779B97F4A7C15ull) ^ a.perturb_seed) % 8 == 0) {  // test hook
            const uint64_t t0 = global_ns();
            while (global_ns() - t0 < a.perturb_ns) __nanosleep(200);
          }
          IO::write(L.tagg, k, IO::GW, epoch, kPartial, agg);  // compact: tile k at k * ST words
          if (tr) tr[uint64_t(k) * 8 + 3] = global_ns();
        });
    // the last tile of a group publishes the group aggregate (warp 1: it polls
    // the group's other 31 aggregates, published by lower tickets)
    if (k % kLagGroup == kLagGroup - 1 && warp == 1) {
      const uint64_t grp = k / kLagGroup;
      C v{};
      bool ok = lane == kWarp - 1;
      if (ok) v = s_carry_agg;  // this tile's own aggregate
      while (true) {
        if (!ok) {
          uint64_t raw[ST];
          const uint64_t* p = L.tagg + (grp * kLagGroup + lane) * ST;
#pragma unroll
          for (int i = 0; i < ST; i += 2) {
            if constexpr (ST == 1) raw[0] = ld_relaxed_gpu(p);
            else ld_relaxed_gpu_v2(p + i, raw[i], raw[i + 1]);
          }
          ok = IO::decode(raw, epoch, v, a.epoch_mask) != 0;
        }
        if (__all_sync(kFullMask, ok)) break;
      }
      Opt<C> x{v, true};
#pragma unroll
      for (unsigned d = 1; d < kWarp; d <<= 1) {
        Opt<C> got{shfl_down(x.v, d), __shfl_down_sync(kFullMask, int(x.has), d) != 0};
        if (lane + d < kWarp) x = opt_combine(cop, x, got);
      }
      if (lane == 0) IO::write(L.gstate, grp, IO::GW, epoch, kPartial, x.v);
    }
  }
  __syncthreads();  // every read of A's tile is done (and s_carry / s_self_agg are visible)
  if (!hasB) return;

  // ---- B: re-load tile j (L2), fold it, compose with the carry, emit, store
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bar, kSmemTileBytes);
    tma_load_2d_hint(buf, &tmap, 0, int(j) * kScanThreads, &bar, l2_policy_evict_first());
  }
  mbar_wait(&bar, phase);
  if (tr && threadIdx.x == 0) tr[uint64_t(k) * 8 + 5] = global_ns();
  const Opt<A> row_ex = tile_row_prefix(std::true_type{}, std::true_type{}, [](const A&) {});
  const Opt<C> carry = s_carry;
  if (threadIdx.x == 0 && (j % kLagGroup == kLagGroup - 1 || j == a.ntiles - 1)) {
    const C agg = s_self_agg;  // tile j's aggregate (A(j)'s, read by the look-back)
    const C pre = carry.has ? cop(carry.v, agg) : agg;
    if (j % kLagGroup == kLagGroup - 1) IO::write(L.gstate, j / kLagGroup, IO::GW, epoch, kPrefix, pre);
    if (j == a.ntiles - 1 && a.total_out) *a.total_out = M::CT::to_s(pre);
  }
  const Opt<A> tile_ex = carry.has ? Opt<A>{M::from_c(carry.v), true} : Opt<A>{A{}, false};
  const Opt<A> run = opt_combine(aop, tile_ex, row_ex);
  using E = std::conditional_t<M::kNarrowEmit, S, A>;
  Opt<E> em;
  if constexpr (M::kNarrowEmit)
    em = Opt<E>{M::lower(run.v), run.has};
  else
    em = run;
  // the running value is present for every row but the global first one:
  // the per-element has-checks (selects) only run in that row
  auto emit_rows = [&](auto has_tag) {
    constexpr bool kHas = decltype(has_tag)::value;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 v = lds128(buf + swz128(threadIdx.x, c));
      T x[EPC];
      memcpy(x, &v, 16);
      S o[EPC];
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        E y;
        if constexpr (M::kNarrowEmit) y = a.f(x[e]);
        else y = M::lift(a.f(x[e]));
        auto eop = [&](const E& p, const E& q) {
          if constexpr (M::kNarrowEmit) return a.op(p, q);
          else return aop(p, q);
        };
        auto elower = [&](const E& w) {
          if constexpr (M::kNarrowEmit) return w;
          else return M::lower(w);
        };
        if constexpr (kHas) {
          if constexpr (Inclusive) {
            em.v = eop(em.v, y);
            o[e] = elower(em.v);
          } else {
            o[e] = elower(em.v);
            em.v = eop(em.v, y);
          }
        } else if constexpr (Inclusive) {
          em.v = em.has ? eop(em.v, y) : y;
          em.has = true;
          o[e] = elower(em.v);
        } else {
          o[e] = em.has ? elower(em.v) : a.identity;
          em.v = em.has ? eop(em.v, y) : y;
          em.has = true;
        }
      }
      uint4 w;
      memcpy(&w, o, 16);
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(buf + swz128(threadIdx.x, c))),
                   "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                   : "memory");
    }
  };
  if (em.has)
    emit_rows(std::true_type{});
  else
    emit_rows(std::false_type{});
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (tr) tr[uint64_t(k) * 8 + 6] = global_ns();
    tma_store_2d_hint(&tmap_out, 0, int(j) * kScanThreads, buf, l2_policy_evict_first());
    tma_store_commit();
    tma_store_wait_read();
    if (tr) tr[uint64_t(k) * 8 + 7] = global_ns();
  }

}


// ---------------------------------------------------------------------------
// Workspace + launch.

// Workspace: [256-byte control block (ticket, epoch) | one slot per group of
// P tile states (TileStateIO)].  Full-speed slots are 256 bytes (kSlotWords,
// DESIGN.md §4); a smaller workspace is accepted down to packed groups
// (kMinSlotWords = one 32-byte group) at some look-back speed.  The size
// depends on S only, so a workspace made for S (make_scan_workspace<S>) fits
// every T: the bound is the larger of the general kernel's tiles (256 x 64
// bytes of S) at packed groups and the smem kernel's tiles of a
// sizeof(S)-byte T at full slots.
template <class T, class S, class Op>
struct ScanWs {
  using C = typename CarryTraits<S, Op>::C;
  using IO = TileStateIO<C>;
  static constexpr uint64_t kTileGeneral = uint64_t(kScanThreads) * scan_items<S>();
  static constexpr uint32_t kMinSlotWords = uint32_t(IO::GW);
  static constexpr uint32_t kSlotWords = kMinSlotWords > kStateSlotWords ? kMinSlotWords : kStateSlotWords;
  static constexpr uint64_t kSizedTile =  // smem tile of a T with sizeof(T) == sizeof(S)
      sizeof(S) >= 16 ? 2 * uint64_t(kScanThreads) * (kRowBytes / 16)
                      : uint64_t(kScanThreads) * (sizeof(S) <= uint64_t(kRowBytes) ? kRowBytes / sizeof(S) : 1);
  static uint64_t min_bytes_for(uint64_t tiles) { return 256 + IO::slots(tiles ? tiles : 1) * kMinSlotWords * 8; }
  // full-speed bytes for n items: the single-pass kernels' states, or the
  // lagged kernel's layout (LagWs) when it takes the scan, whichever is larger
  static uint64_t bytes(uint64_t n);
  static uint64_t base_bytes(uint64_t n) {
    const uint64_t full = 256 + IO::slots(n ? ceil_div(n, kSizedTile) : 1) * kSlotWords * 8;
    const uint64_t packed = min_bytes_for(ceil_div(n, kTileGeneral));
    return full > packed ? full : packed;
  }
  // Largest slot stride (64-bit words, power of two, <= kSlotWords) that fits
  // the groups of `tiles` tiles in `ws_bytes`; 0 when even packed groups do not fit.
  static uint32_t slot_words(uint64_t tiles, uint64_t ws_bytes) {
    for (uint32_t w = kSlotWords; w >= kMinSlotWords && w > 0; w >>= 1)
      if (256 + IO::slots(tiles ? tiles : 1) * uint64_t(w) * 8 <= ws_bytes) return w;
    return 0;
  }
  static uint64_t claim_bytes(uint64_t tiles, uint32_t stride) { return 256 + IO::slots(tiles) * stride * 8; }
};

#ifndef FORGE_SCAN_LAG_MAX_T
// largest element (bytes) taken by the lagged scan.  16-byte elements (Mat2)
// take the single-pass kernel since its tiles are blockIdx-ordered: Mat2 2^27
// 5,759-5,823 GB/s single-pass vs 5,574-5,618 lagged (tools/probe_order.py,
// profiles/r02/probe_order_single_pass_all_session5.log); 8-byte elements with
// 16-byte carries (f32 affine, f64 carry) keep the lagged kernel (5,624-5,643
// vs 5,605).
#define FORGE_SCAN_LAG_MAX_T 8
#endif

// Lagged-scan workspace: [256-byte control block | tile
// aggregates | group states | full-tile total | tail sub-workspace].
template <class T, class S, class Op>
struct LagWs {
  using C = typename CarryTraits<S, Op>::C;
  using A = typename ScanMath<S, Op>::A;
  static constexpr uint64_t ST = uint64_t(TileStateIO<C>::STRIDE);
  static constexpr uint64_t align(uint64_t v) { return (v + 255) & ~uint64_t(255); }
  static uint64_t tagg_off(uint64_t) { return 256; }
  static uint64_t gstate_off(uint64_t tiles) { return tagg_off(tiles) + align(tiles * ST * 8); }
  static uint64_t total_off(uint64_t tiles) { return gstate_off(tiles) + align(ceil_div(tiles, kLagGroup) * ST * 8); }
  static uint64_t tail_off(uint64_t tiles) { return total_off(tiles) + 256; }
  // the tail launch (< one tile) never takes the lagged kernel
  static uint64_t bytes(uint64_t tiles, uint64_t tile_items) {
    return tail_off(tiles) + ScanWs<T, S, Op>::base_bytes(tile_items);
  }
};

// The lagged kernel takes 16-byte carries (f64 affine, Mat2); for carries of
// at most 8 bytes the single-pass kernel is as fast or faster since the claim
// became relaxed and the tile an L2 prefetch (2^28 / 2^27, GB/s, single-pass
// vs lagged): f32 sum 5,870 / 5,900, f64 sum 5,727 / 5,690, i32 sum 5,933 /
// 5,818, i32 max 5,951 / 5,790, i64 sum 5,888 / 5,689, argmax 5,490 / 5,424
// (with the row-prefix ring), affine 5,414 / 5,605, Mat2 5,419 /
// 5,606.  32-byte carries (quaternion) spill at 6 CTAs/SM.
template <class T, class S, class Op>
constexpr bool lag_scan_type_ok() {
  return smem_scan_type_ok<T>() && sizeof(S) == sizeof(T) && sizeof(T) <= FORGE_SCAN_LAG_MAX_T &&
         sizeof(typename CarryTraits<S, Op>::C) > 8 && sizeof(typename CarryTraits<S, Op>::C) <= 16;
}


// Development knobs (FORGE_DEV builds only; constants otherwise).
inline uint32_t scan_lookback_mode() {
  static const uint32_t v = dev_knob("FORGE_SCAN_LOOKBACK", 0);
  return v;
}
inline uint32_t scan_backoff_ns() {
  static const uint32_t v = dev_knob("FORGE_SCAN_BACKOFF_NS", 0);
  return v;
}
inline bool scan_force_regs() {
  static const bool v = dev_knob("FORGE_SCAN_REGS", 0) != 0;
  return v;
}
// Lag D of the lagged scan (scan_lag_kernel), in tiles; 0 = the single-pass
// kernel.  Measured on B200 (148 SMs, f32 / i32 / affine / argmax / Mat2 at
// 2^28, GB/s, relaxed claims, row-prefix ring for argmax — all five took the
// lagged kernel then): D = 384: 4945 /
// 4496 / 4385 / 4209 / 4305 (B waits for A's aggregates); 448: 5399 / 4923 /
// 4841 / 4483 / 4852; 518: 5572 / 5344 / 5162 / 4915 / 5150; 600: 5600 / 5486
// / 5246 / 4968 / 5266; 680: 5571 / 5497 / 5208 / 4972 / 5226; 760: 5484 /
// 5397 / 5113 / 4950 / 5130; 1000: 4918 / 4895 / 4836 / 4679 / 4830 (the
// re-read starts missing L2).  D scales with the resident tiles: 4 per SM.
inline uint32_t scan_lag() {
  static const uint32_t v = dev_knob("FORGE_SCAN_LAG", device_props().sm_count * 4);
  return v;
}
// L2 prefetch distance of the single-pass tile kernel, in tiles: CTA g
// prefetches tile g + ahead, so the tile a CTA claims is in L2 before the
// claim returns.  Measured (2^28, GB/s, f32 / i32 / argmax): ahead 0 (the
// CTA's own tile): 5,880 / 5,950 / 5,472; 100: 6,054 / 6,161 / 5,574; 200:
// 6,054-6,089 / 6,161 / 5,574; 300: 6,054-6,089 / 6,160 / 5,574; 600: 5,823 /
// 5,883 / 5,516; 900: 4,850 / 4,850 / 5,045 (the prefetched tiles start to be
// evicted before use) — one tile per SM.  The lagged kernel keeps 0 (its L2
// already holds the D-tile re-read window: affine 5,620 at 0 and 100, 5,575
// at 300, 4,950 at 600).
inline uint32_t scan_prefetch_ahead() {
  static const uint32_t v = dev_knob("FORGE_SCAN_PREFETCH_AHEAD", device_props().sm_count);
  return v;
}
// Tile order of the single-pass tile kernel: 1 = blockIdx.x (default): the
// tile's TMA load is issued at CTA start and the claim — still made, for the
// launch epoch and the ticket reset — overlaps it; forward progress relies on
// the hardware dispatching a launch's CTAs in increasing blockIdx order, as
// CUB's single-pass scan (tile_idx = blockIdx.x) does.  0 = tickets (tile =
// claim order, deadlock-free under any dispatch order; FORGE_DEV knob).
// Measured 2^28 (GB/s, tickets -> blockIdx): f32 6,053 -> 6,160-6,197, i32
// 6,159 -> 6,272-6,306, argmax 5,560-5,612 -> 5,726-5,790, i64 6,059 -> 6,237;
// 2^23 f32 3,549 -> 3,560-3,972 (tools/probe_order.py).
inline uint32_t scan_block_order() {
  static const uint32_t v = dev_knob("FORGE_SCAN_BLOCK_ORDER", 1);
  return v;
}
// The lagged kernel keeps tickets: with ticket = blockIdx.x (A's load before
// the claim) it measured slower, affine 2^28 5,624-5,643 -> 5,472-5,501 GB/s,
// Mat2 2^27 5,574-5,618 -> 5,374-5,458 (tools/probe_order.py).
inline uint32_t scan_lag_block_order() {
  static const uint32_t v = dev_knob("FORGE_SCAN_LAG_BLOCK_ORDER", 0);
  return v;
}
// Prefetch distance of the blockIdx-ordered single-pass kernel (its own tile
// is TMA-loaded at CTA start; the prefetch serves the CTAs of later waves):
// measured 2^28 (GB/s) at 0 / 1 / 2 / 3 tiles per SM: f32 5,695 / 6,199-6,201
// / 6,237 / 6,236, i32 5,633 / 6,310-6,313 / 6,383 / 6,382, i64 5,757 /
// 6,240-6,258 / 6,299 / 6,314, argmax 5,249 / 5,742 / 5,743 / 5,743, Mat2
// (64 KB tiles) 5,308 / 5,759-5,774 / 5,774 / 5,307 — two tiles per SM.
inline uint32_t scan_block_prefetch_ahead() {
  static const uint32_t v = dev_knob("FORGE_SCAN_BLOCK_PREFETCH_AHEAD", 2 * device_props().sm_count);
  return v;
}
inline bool scan_no_tma_store() {
  static const bool v = dev_knob("FORGE_SCAN_NO_TMA_STORE", 0) != 0;
  return v;
}

// 32 KB sub-tiles per CTA tile of the default kernel: measured (f32 / i32 /
// affine / argmax / Mat2 at 2^28, GB/s) R=1: 4896 / 4941 / 3747 / 4612 / 3801,
// R=2: 4635 / 4658 / 3491 / 4264 / 4532 — so R = 2 for 16-byte elements only.
template <class T>
constexpr int scan_subtiles() {
  return sizeof(T) >= 16 ? 2 : 1;
}

template <class T, class S, class F, class Op, bool Inclusive, int R>
cudaError_t launch_scan_smem(const ScanArgs<T, S, F, Op>& a, const CUtensorMap& tmap, const CUtensorMap& tmap_out,
                             bool tstore, cudaStream_t stream) {
  auto kern = scan_smem_kernel<T, S, F, Op, Inclusive, R>;
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(scan_smem_dyn(R)));
    // Maximum shared-memory carveout: residency (tiles in flight) is what
    // hides the look-back latency; the kernel barely uses L1.
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done_dev = dev;
  }
  kern<<<a.ntiles, kScanThreads, scan_smem_dyn(R), stream>>>(a, tmap, tmap_out, tstore);
  return cudaGetLastError();
}

#ifdef FORGE_DEV
// Per-tile phase timestamps (tools/trace_scan.py): a buffer of its own, never
// the caller's workspace.  8 words per tile; fetched with forge_dev_scan_trace.
inline uint64_t*& scan_trace_buffer() {
  static uint64_t* p = nullptr;
  return p;
}
inline uint64_t& scan_trace_words() {
  static uint64_t w = 0;
  return w;
}
inline uint64_t* scan_trace_for(uint64_t tiles) {
  if (!dev_knob("FORGE_SCAN_TRACE", 0)) return nullptr;
  if (scan_trace_words() < tiles * 8) {
    if (scan_trace_buffer()) cudaFree(scan_trace_buffer());
    scan_trace_buffer() = nullptr;
    if (cudaMalloc(&scan_trace_buffer(), tiles * 64) != cudaSuccess) return nullptr;
    scan_trace_words() = tiles * 8;
  }
  return scan_trace_buffer();
}
#endif

// The lagged kernel takes contiguous scans of >= lag_min_tiles() full tiles
// (below ~3 lags the single-pass kernel is faster: CUDA-graph f32 2^20 6.4 vs
// 11.3 us, 2^23 18.3 vs 19.6, 2^24 39.3 vs 37.1, 2^26 120 vs 113).
inline uint64_t lag_min_tiles() {
  const uint64_t d = scan_lag();
  return d ? (3 * d > 4 * kLagGroup ? 3 * d : 4 * kLagGroup) : ~uint64_t(0);
}

template <class T, class S, class Op>
uint64_t ScanWs<T, S, Op>::bytes(uint64_t n) {
  uint64_t b = base_bytes(n);
  if constexpr (lag_scan_type_ok<T, S, Op>()) {
    constexpr uint64_t kTile = uint64_t(kScanThreads) * smem_scan_items<T>();
    const uint64_t tiles = n / kTile;
    if (tiles >= lag_min_tiles()) {
      const uint64_t lag = LagWs<T, S, Op>::bytes(tiles, kTile);
      b = lag > b ? lag : b;
    }
  }
  return b;
}

// Launch.  `ws` holds `ws_bytes` bytes (>= ScanWs::min_bytes_for(tiles) of the
// kernel that runs; ScanWs::bytes(n) gives full-speed slots), zeroed once at
// creation.  Returns cudaErrorInvalidValue when the workspace is too small
// (callers check first and raise WorkspaceTooSmall).
// `hooks`: test-only ablation / schedule perturbation (ScanTestHooks).
template <class T, class S, class F, class Op>
cudaError_t launch_scan(const T* src, uint64_t src_stride, S* dst, uint64_t dst_stride, uint64_t n,
                        bool inclusive, const F& f, const Op& op, const S& identity,
                        const S* carry_in, S* total_out, void* ws, uint64_t ws_bytes, cudaStream_t stream,
                        const ScanTestHooks& hooks = {}) {
  using WsT = ScanWs<T, S, Op>;
  if (n == 0) return cudaSuccess;
  if (ceil_div(n, WsT::kTileGeneral) >= (1ull << 31)) return cudaErrorInvalidValue;
  ScanArgs<T, S, F, Op> a{src,      dst,      n,         src_stride, dst_stride,
                          f,        op,       identity,  carry_in,   total_out,
                          reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + 256),
                          static_cast<uint32_t*>(ws), 0u, 0u, scan_lookback_mode(), nullptr,
                          scan_backoff_ns(), hooks.relax_epoch ? 0u : 0x3fffffffu, hooks.perturb_seed,
                          hooks.perturb_ns,
                          scan_block_order() ? scan_block_prefetch_ahead() : scan_prefetch_ahead(),
                          scan_block_order()};
  // The TMA tile kernel is instantiated only for power-of-two element sizes
  // up to 16 bytes (whole items per 16-byte chunk); other types take the
  // register kernel.
  // lagged scan: 16-byte carries (lag_scan_type_ok)
  if constexpr (lag_scan_type_ok<T, S, Op>()) {
    if (const uint32_t lag = scan_lag(); lag && src_stride == 1 && dst_stride == 1) {
      constexpr uint64_t kTile = uint64_t(kScanThreads) * smem_scan_items<T>();
      using LW = LagWs<T, S, Op>;
      const uint64_t nfull = n / kTile;
      const uint64_t tail = n - nfull * kTile;
      CUtensorMap tin, tout;
      if (nfull >= lag_min_tiles() && nfull + lag < (1ull << 30) &&
          ws_bytes >= LW::bytes(nfull, kTile) &&
          make_rows128_map(&tin, src, nfull * kTile * sizeof(T) / kRowBytes, uint32_t(kScanThreads)) &&
          make_rows128_map(&tout, dst, nfull * kTile * sizeof(S) / kRowBytes, uint32_t(kScanThreads))) {
        char* w = static_cast<char*>(ws);
        LagArgs<T, S, F, Op> L{a,
                               reinterpret_cast<uint64_t*>(w + LW::tagg_off(nfull)),
                               reinterpret_cast<uint64_t*>(w + LW::gstate_off(nfull)),
                               lag,
                               uint32_t(nfull + lag)};
        L.s.ntiles = uint32_t(nfull);
        L.s.prefetch_ahead = 0;  // scan_prefetch_ahead
        L.s.block_order = scan_lag_block_order();
#ifdef FORGE_DEV
        L.s.trace = scan_trace_for(nfull + lag);
#endif
        S* full_total = reinterpret_cast<S*>(w + LW::total_off(nfull));
        L.s.total_out = tail ? full_total : total_out;
        if (const cudaError_t e = ws_claim(ws, kWsTagScanLag, LW::tail_off(nfull), stream); e != cudaSuccess) return e;
        auto kern = inclusive ? scan_lag_kernel<T, S, F, Op, true> : scan_lag_kernel<T, S, F, Op, false>;
        static thread_local int done_dev = -1;
        int dev = 0;
        cudaGetDevice(&dev);
        if (done_dev != dev) {
          cudaFuncSetAttribute(scan_lag_kernel<T, S, F, Op, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kSmemScanDyn));
          cudaFuncSetAttribute(scan_lag_kernel<T, S, F, Op, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kSmemScanDyn));
          cudaFuncSetAttribute(scan_lag_kernel<T, S, F, Op, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          cudaFuncSetAttribute(scan_lag_kernel<T, S, F, Op, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          done_dev = dev;
        }
        kern<<<uint32_t(nfull + lag), kScanThreads, kSmemScanDyn, stream>>>(L, tin, tout);
        if (const cudaError_t e = cudaGetLastError(); e != cudaSuccess || !tail) return e;
        // the partial last tile: a tail launch seeded with the full tiles' total
        const uint64_t off = nfull * kTile;
        return launch_scan<T, S, F, Op>(src + off, 1, dst + off, 1, tail, inclusive, f, op, identity, full_total,
                                        total_out, w + LW::tail_off(nfull), ws_bytes - LW::tail_off(nfull), stream,
                                        hooks);
      }
    }
  }
  if constexpr (smem_scan_type_ok<T>()) {
    constexpr int R = scan_subtiles<T>();
    constexpr uint64_t kTile = uint64_t(R) * kScanThreads * smem_scan_items<T>();
    CUtensorMap tmap;
    const bool smem = !scan_force_regs() && src_stride == 1 && dst_stride == 1 && n >= kTile &&
                      make_rows128_map(&tmap, src, (n * sizeof(T)) / kRowBytes, uint32_t(kScanThreads));
    if (smem) {
      a.ntiles = uint32_t(ceil_div(n, kTile));
      a.state_stride = WsT::slot_words(a.ntiles, ws_bytes);
      if (a.state_stride == 0) return cudaErrorInvalidValue;
#ifdef FORGE_DEV
      a.trace = scan_trace_for(a.ntiles);
#endif
      if (const cudaError_t e = ws_claim(ws, kWsTagScan, WsT::claim_bytes(a.ntiles, a.state_stride), stream);
          e != cudaSuccess)
        return e;
      CUtensorMap tmap_out = tmap;
      const bool tstore = sizeof(S) == sizeof(T) && !scan_no_tma_store() &&
                          make_rows128_map(&tmap_out, dst, (n * sizeof(S)) / kRowBytes, uint32_t(kScanThreads));
      return inclusive ? launch_scan_smem<T, S, F, Op, true, R>(a, tmap, tmap_out, tstore, stream)
                       : launch_scan_smem<T, S, F, Op, false, R>(a, tmap, tmap_out, tstore, stream);
    }
  }
  a.ntiles = uint32_t(ceil_div(n, WsT::kTileGeneral));
  a.state_stride = WsT::slot_words(a.ntiles, ws_bytes);
  if (a.state_stride == 0) return cudaErrorInvalidValue;
  if (const cudaError_t e = ws_claim(ws, kWsTagScan, WsT::claim_bytes(a.ntiles, a.state_stride), stream);
      e != cudaSuccess)
    return e;
  if (inclusive)
    scan_kernel<T, S, F, Op, true><<<a.ntiles, kScanThreads, 0, stream>>>(a);
  else
    scan_kernel<T, S, F, Op, false><<<a.ntiles, kScanThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace forge::cuda
