// forge/cuda/scan_cyclic.cuh — sharded scan with a CROSS-GPU decoupled
// look-back.
//
// The global array is cut into chunks of TPC tiles; chunk c lives on shard
// c mod G (block-cyclic), each shard holding its chunks back to back.  Every
// shard runs the single-pass protocol of scan.cuh (ticketed tiles in local
// order, tile aggregate published as PARTIAL, look-back to the nearest PREFIX,
// own PREFIX published, outputs emitted from the smem tile) — but the tile
// states of global tile T live on T's OWNER, and a look-back that crosses a
// chunk boundary reads the previous chunk's states on the previous shard:
// peer memory over NVLink / NVSwitch (`ld.relaxed.sys` / `st.relaxed.sys`),
// no collective, no host step.  Each shard reads its n/G input and writes its
// n/G output ONCE: 2n/G HBM bytes per GPU against reduce-then-scan's 3n/G
// (sharded.py / forge_sharded_scan), at the price of a pipeline skew of about
// one chunk per shard at the start.
//
// Progress: every tile waits only on tiles of LOWER global index; each shard
// claims its tiles in local (= global) order, so the lowest unfinished tile
// is always claimed or claimable and all its predecessors are done.  The
// EMULATED form (all shards on one GPU, one launch, tickets dealt round-robin
// to the virtual shards) needs the stronger bound TPC * G <= resident CTAs,
// checked at launch (a tile may wait on a higher ticket of the previous
// virtual shard, at most TPC * G tickets ahead).
#pragma once

#include "forge/cuda/scan.cuh"

namespace forge::cuda {

constexpr int kCyclicMaxShards = 8;  // virtual shards per launch (emulation); tensor maps per launch

__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t r;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct CyclicMaps {
  CUtensorMap in[kCyclicMaxShards];
  CUtensorMap out[kCyclicMaxShards];
};

template <class T, class S, class F, class Op>
struct CyclicArgs {
  const T* src[kCyclicMaxShards];  // per virtual shard of this launch
  S* dst[kCyclicMaxShards];
  uint64_t local_n[kCyclicMaxShards];   // elements held by the shard
  uint32_t local_tiles[kCyclicMaxShards];
  uint64_t* states[kCyclicMaxShards];  // tile states of EVERY shard (by rank; peer pointers across GPUs)
  uint32_t* ctrl;                       // this launch's ticket word (reset by the last claimer)
  uint32_t epoch;                       // from the host: process-wide monotonic, never 0 — the
                                        // shards' kernels agree on it without reading each other
  uint64_t n;                           // global length
  uint64_t tiles;                       // global tiles
  uint32_t tpc;                         // tiles per chunk
  uint32_t G;                           // shards in the group
  uint32_t rank0, nvirt;                // virtual shard v of this launch is rank rank0 + v
  uint32_t nclaims;                     // sum of local_tiles over this launch's virtual shards
  uint32_t stride;                      // 64-bit words per tile state slot
  uint32_t prefetch_ahead;              // CTA g L2-prefetches ticket g + this's tile (launch_scan_cyclic)
  F f;
  Op op;
  S identity;
};

// Global tile T -> (owner rank, local tile index).
__host__ __device__ __forceinline__ void cyclic_locate(uint64_t T, uint32_t tpc, uint32_t G, uint32_t& owner,
                                                       uint64_t& local) {
  const uint64_t c = T / tpc;
  owner = uint32_t(c % G);
  local = (c / G) * tpc + T % tpc;
}

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads, 6)
    scan_cyclic_kernel(const CyclicArgs<T, S, F, Op> a, const __grid_constant__ CyclicMaps maps) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  constexpr int SW = IO::SW;
  constexpr int ST = IO::STRIDE;
  constexpr int IT = smem_scan_items<T>();
  constexpr int EPC = 16 / int(sizeof(T));
  constexpr int NCH = kRowBytes / 16;
  constexpr int NW = kScanThreads / kWarp;
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_q;
  __shared__ Opt<A> s_warp[NW];
  __shared__ Opt<A> s_carry;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };
  unsigned char* buf =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;

  // ---- claim: ticket q -> virtual shard v = q % nvirt, its local tile q / nvirt
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    // L2 prefetch of ticket blockIdx.x + ahead's tile while the claim is in
    // flight (scan.cuh scan_prefetch_ahead); the first `ahead` CTAs also
    // prefetch their own guessed tile
    auto prefetch = [&](uint64_t q) {
      const uint32_t gv = uint32_t(q % a.nvirt);
      const uint64_t gl = q / a.nvirt;
      if (gl < a.local_tiles[gv] && (gl + 1) * kTile <= a.local_n[gv])
        tma_prefetch_2d_hint(&maps.in[gv], 0, int(gl) * kScanThreads, l2_policy_evict_normal());
    };
    if (blockIdx.x < a.prefetch_ahead || a.prefetch_ahead == 0) prefetch(blockIdx.x);
    if (a.prefetch_ahead) prefetch(uint64_t(blockIdx.x) + a.prefetch_ahead);
    const uint32_t q = atom_add_relaxed_gpu(a.ctrl, 1u);  // orders nothing (states carry the epoch)
    if (q == a.nclaims - 1) st_relaxed_gpu(a.ctrl, 0u);
    s_q = q;
  }
  __syncthreads();
  // tickets beyond a short virtual shard's tiles are skipped (round-robin deal)
  const uint32_t q = s_q, epoch = a.epoch;
  const uint32_t v = q % a.nvirt;
  const uint64_t l = q / a.nvirt;
  if (l >= a.local_tiles[v]) return;
  const uint32_t rank = a.rank0 + v;
  const uint64_t chunk = (l / a.tpc) * a.G + rank;
  const uint64_t Tg = chunk * a.tpc + l % a.tpc;  // global tile
  const uint64_t lbase = l * kTile;               // local element offset
  const T* src = a.src[v];
  S* dst = a.dst[v];
  const bool full = lbase + kTile <= a.local_n[v];
  if (full && threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, kSmemTileBytes);
    tma_load_2d(buf, &maps.in[v], 0, int(l) * kScanThreads, &bar);
  }
  const uint64_t base = lbase + uint64_t(threadIdx.x) * IT;
  const uint64_t avail = base < a.local_n[v] ? a.local_n[v] - base : 0;
  const int count = full ? IT : (avail >= uint64_t(IT) ? IT : int(avail));

  // ---- pass 1: row totals
  Opt<A> tot{A{}, false};
  if (full) {
    mbar_wait(&bar, 0);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 w = lds128(buf + swz128(threadIdx.x, c));
      T x[EPC];
      memcpy(x, &w, 16);
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const A y = M::lift(a.f(x[e]));
        tot.v = (c == 0 && e == 0) ? y : aop(tot.v, y);
      }
    }
    tot.has = true;
  } else {
    for (int k = 0; k < count; ++k) {
      const A y = M::lift(a.f(src[base + k]));
      tot.v = k == 0 ? y : aop(tot.v, y);
    }
    tot.has = count > 0;
  }
  // block scan of the row totals
  Opt<A> incl = warp_scan_incl(aop, tot);
  if (lane == kWarp - 1) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    Opt<A> w = lane < NW ? s_warp[lane] : Opt<A>{A{}, false};
    w = warp_scan_incl(aop, w);
    if (lane < NW) s_warp[lane] = w;
  }
  __syncthreads();
  const Opt<A> agg = s_warp[NW - 1];

  // ---- publish + cross-shard decoupled look-back
  auto write_state = [&](uint64_t* p, uint32_t kind, const C& val) {
    Words<C> wd = to_words(val);
    const uint64_t hi = uint64_t((epoch << 2) | kind) << 32;
#pragma unroll
    for (int i = 0; i < ST; ++i) st_relaxed_sys(p + i, hi | (i < SW ? wd.w[i] : 0u));
  };
  uint64_t* mine = a.states[rank] + l * a.stride;
  if (Tg == 0) {
    if (threadIdx.x == 0) {
      write_state(mine, kPrefix, M::to_c(agg.v));
      s_carry = Opt<A>{A{}, false};
    }
  } else {
    const C agg_c = M::to_c(agg.v);
    if (threadIdx.x == 0) write_state(mine, kPartial, agg_c);
    if (warp == 0) {
      Opt<C> carry{C{}, false};
      int64_t hi = int64_t(Tg);  // window: tiles hi-1 .. hi-32
      for (;;) {
        const int64_t P = hi - 1 - int64_t(lane);
        uint32_t kind = P < 0 ? 4u : 0u;
        C val{};
        const uint64_t* sp = nullptr;
        if (P >= 0) {
          uint32_t own;
          uint64_t loc;
          cyclic_locate(uint64_t(P), a.tpc, a.G, own, loc);
          sp = a.states[own] + loc * a.stride;
        }
        for (;;) {
          if (kind == 0) {
            uint64_t raw[ST];
#pragma unroll
            for (int i = 0; i < ST; ++i) raw[i] = ld_relaxed_sys(sp + i);
            kind = IO::decode(raw, epoch, val);
          }
          if (__all_sync(kFullMask, kind != 0)) break;
        }
        const unsigned pm = __ballot_sync(kFullMask, kind == kPrefix);
        const int near = pm ? __ffs(int(pm)) - 1 : kWarp;
        Opt<C> x{val, int(lane) <= near && kind != 4u};
#pragma unroll
        for (unsigned d = 1; d < kWarp; d <<= 1) {  // older (higher lane) on the left
          Opt<C> got{shfl_down(x.v, d), __shfl_down_sync(kFullMask, int(x.has), d) != 0};
          if (lane + d < kWarp) x = opt_combine(cop, got, x);
        }
        carry = opt_combine(cop, shfl_idx_opt(x, 0), carry);
        if (near < kWarp || hi <= int64_t(kWarp)) break;
        hi -= kWarp;
      }
      if (lane == 0) {
        write_state(mine, kPrefix, cop(carry.v, agg_c));
        s_carry = Opt<A>{M::from_c(carry.v), true};
      }
    }
  }
  __syncthreads();

  // ---- pass 2: running prefixes
  Opt<A> run;
  {
    const Opt<A> warp_ex = warp > 0 ? s_warp[warp - 1] : Opt<A>{A{}, false};
    Opt<A> lane_ex = shfl_up_opt(incl, 1);
    if (lane == 0) lane_ex.has = false;
    run = opt_combine(aop, opt_combine(aop, s_carry, warp_ex), lane_ex);
  }
  if (full) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 w = lds128(buf + swz128(threadIdx.x, c));
      T x[EPC];
      memcpy(x, &w, 16);
      S o[EPC];
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const A y = M::lift(a.f(x[e]));
        if constexpr (Inclusive) {
          run.v = run.has ? aop(run.v, y) : y;
          run.has = true;
          o[e] = M::lower(run.v);
        } else {
          o[e] = run.has ? M::lower(run.v) : a.identity;
          run.v = run.has ? aop(run.v, y) : y;
          run.has = true;
        }
      }
      uint4 wo;
      memcpy(&wo, o, 16);
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(buf + swz128(threadIdx.x, c))),
                   "r"(wo.x), "r"(wo.y), "r"(wo.z), "r"(wo.w)
                   : "memory");
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_2d(&maps.out[v], 0, int(l) * kScanThreads, buf);
      tma_store_commit();
      tma_store_wait_read();
    }
  } else {
    for (int k = 0; k < count; ++k) {
      const A y = M::lift(a.f(src[base + k]));
      if constexpr (Inclusive) {
        run.v = run.has ? aop(run.v, y) : y;
        run.has = true;
        dst[base + k] = M::lower(run.v);
      } else {
        dst[base + k] = run.has ? M::lower(run.v) : a.identity;
        run.v = run.has ? aop(run.v, y) : y;
        run.has = true;
      }
    }
  }
}

// Elements of a length-n global array held by shard `rank` of G under chunks
// of `chunk` elements (chunk c on shard c mod G).
__host__ __device__ inline uint64_t cyclic_local_n(uint64_t n, uint64_t chunk, uint32_t rank, uint32_t G) {
  const uint64_t full = n / chunk, rem = n % chunk;
  uint64_t k = full / G + (rank < full % G ? 1 : 0);
  uint64_t r = k * chunk;
  if (rem && full % G == rank) r += rem;
  return r;
}

template <class T>
constexpr uint64_t cyclic_tile_elems() {
  return uint64_t(kScanThreads) * smem_scan_items<T>();
}

// Workspace per shard: [{epoch, ticket} | one state slot (stride words) per local tile].
template <class S, class Op>
constexpr uint32_t cyclic_stride() {
  using C = typename CarryTraits<S, Op>::C;
  return uint32_t(TileStateIO<C>::STRIDE) > 4 ? uint32_t(TileStateIO<C>::STRIDE) : 4u;  // >= 32 bytes
}

template <class T, class S, class Op>
uint64_t cyclic_ws_bytes(uint64_t local_n) {
  const uint64_t tiles = ceil_div(local_n, cyclic_tile_elems<T>());
  return 256 + (tiles ? tiles : 1) * cyclic_stride<S, Op>() * 8;
}

// One launch over `nvirt` virtual shards (ranks rank0 .. rank0 + nvirt - 1).
template <class T, class S, class F, class Op>
cudaError_t launch_scan_cyclic(CyclicArgs<T, S, F, Op> a, bool inclusive, cudaStream_t stream) {
  constexpr uint64_t kTile = cyclic_tile_elems<T>();
  CyclicMaps maps;
  uint32_t claims = 0;
  uint32_t maxtiles = 0;
  for (uint32_t v = 0; v < a.nvirt; ++v) {
    const uint64_t tiles = ceil_div(a.local_n[v], kTile);
    a.local_tiles[v] = uint32_t(tiles);
    if (tiles > maxtiles) maxtiles = uint32_t(tiles);
    const uint64_t full_rows = (a.local_n[v] / kTile) * kTile * sizeof(T) / kRowBytes;
    if (full_rows && (!make_rows128_map(&maps.in[v], a.src[v], full_rows, uint32_t(kScanThreads)) ||
                      !make_rows128_map(&maps.out[v], a.dst[v], full_rows, uint32_t(kScanThreads))))
      return cudaErrorInvalidValue;
  }
  claims = maxtiles * a.nvirt;  // round-robin deal: every virtual shard gets maxtiles tickets
  if (claims == 0) return cudaSuccess;
  a.nclaims = claims;
  a.stride = cyclic_stride<S, Op>();
  a.prefetch_ahead = scan_prefetch_ahead();
  auto k1 = scan_cyclic_kernel<T, S, F, Op, true>;
  auto k0 = scan_cyclic_kernel<T, S, F, Op, false>;
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev != dev) {
    for (auto k : {k0, k1}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemScanDyn));
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    done_dev = dev;
  }
  (inclusive ? k1 : k0)<<<claims, kScanThreads, kSmemScanDyn, stream>>>(a, maps);
  return cudaGetLastError();
}

}  // namespace forge::cuda
