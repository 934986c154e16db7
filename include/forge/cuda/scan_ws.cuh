// forge/cuda/scan_ws.cuh — warp-specialised persistent scan kernel.
// Included by forge/cuda/scan.cuh after the shared tile machinery (TileStateIO,
// ScanArgs, ScanMath, TMA helpers); not a standalone header.
#pragma once

namespace forge::cuda {

// ---------------------------------------------------------------------------
// Fast path v4: warp-specialised persistent scan.
//
// Per CTA, with a ring of kWsStages TMA-loaded tiles:
//   warp 8  (producer)   tickets in order; 2-D TMA of each claimed tile.
//   warp 9  (aggregator) as soon as a tile lands: ordered fold of every row
//                        (rows visited in a per-lane rotated order so each
//                        quarter-warp touches 8 distinct bank groups), row
//                        totals to smem, ordered warp fold -> PARTIAL.
//   warp 10 (look-back)  decoupled look-back of each tile (32 lanes x LB polls
//                        per round) -> PREFIX, tile carry to smem.
//   warps 0-7 (consumers) block scan of the row totals, running prefixes
//                        written back into the tile, one TMA tensor store.
// PARTIALs no longer wait behind the consumers' pipeline: they appear one
// fold after the data lands, which removes the head-of-line blocking measured
// on the earlier kernels.  Only the look-back warp waits on other CTAs, and
// only on smaller tiles, so progress needs no co-residency.

constexpr int kWsStages = 3;
constexpr int kWsProducer = kScanThreads / kWarp;       // warp 8
constexpr int kWsAggregator = kWsProducer + 1;          // warp 9
constexpr int kWsLookback = kWsProducer + 2;            // warp 10
constexpr int kWsThreads = kScanThreads + 3 * kWarp;    // 352
constexpr int kWsLookbackPolls = 4;                     // per lane -> window 128

template <class A, class C>
struct WsStage {
  Opt<A> rowtot[kScanThreads];
  C agg;
  Opt<A> carry;
};

template <class S, class Op>
using WsStageOf = WsStage<typename ScanMath<S, Op>::A, typename ScanMath<S, Op>::C>;

template <class T, class S, class Op>
constexpr uint32_t ws_dyn_bytes() {
  return uint32_t(kWsStages) * (kSmemTileBytes + uint32_t(sizeof(WsStageOf<S, Op>))) + 1024;
}

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kWsThreads)
    scan_ws_kernel(const ScanArgs<T, S, F, Op> a, const __grid_constant__ CUtensorMap tmap,
                   const __grid_constant__ CUtensorMap tmap_out, bool tma_store) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  using Stage = WsStageOf<S, Op>;
  constexpr int IT = smem_scan_items<T>();
  constexpr int EPC = 16 / int(sizeof(T));
  constexpr int NCH = kRowBytes / 16;
  constexpr int NW = kScanThreads / kWarp;
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t full[kWsStages], aggd[kWsStages], carried[kWsStages], empty[kWsStages];
  __shared__ uint32_t ring[kWsStages];
  __shared__ uint32_t s_epoch;
  __shared__ Opt<A> s_warp[NW];
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };
  unsigned char* base_mem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  auto tile_mem = [&](int s) { return base_mem + size_t(s) * kSmemTileBytes; };
  Stage* stages = reinterpret_cast<Stage*>(base_mem + size_t(kWsStages) * kSmemTileBytes);
  const bool tail_partial = (a.n % kTile) != 0;
  const unsigned warp = threadIdx.x / kWarp, lane = lane_id();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&aggd[s], 1);
      mbar_init(&carried[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWsProducer) {
    if (lane != 0) return;
    const uint32_t epoch = ld_acquire_gpu(a.ctrl + 2);
    s_epoch = epoch;
    for (uint32_t it = 0;; ++it) {
      const int s = int(it % kWsStages);
      if (it >= uint32_t(kWsStages)) mbar_wait(&empty[s], ((it / kWsStages) - 1) & 1u);
      uint32_t t = atom_add_acq_rel_gpu(a.ctrl + 0, 1u);
      if (t == a.ntiles + gridDim.x - 1) {
        st_relaxed_gpu(a.ctrl + 0, 0u);
        st_relaxed_gpu(a.ctrl + 2, epoch + 1u);
      }
      if (t >= a.ntiles) t = kNoTile;
      ring[s] = t;
      if (t != kNoTile && !(tail_partial && t == a.ntiles - 1)) {
        mbar_arrive_expect_tx(&full[s], kSmemTileBytes);
        tma_load_2d(tile_mem(s), &tmap, 0, int(t) * kScanThreads, &full[s]);
      } else {
        mbar_arrive(&full[s]);
      }
      if (t == kNoTile) return;
    }
  }

  if (warp == kWsAggregator) {
    // lane l owns rows 8l .. 8l+7; at step k it folds row 8l + ((k + l) & 7).
    for (uint32_t it = 0;; ++it) {
      const int s = int(it % kWsStages);
      mbar_wait(&full[s], (it / kWsStages) & 1u);
      const uint32_t tile = ring[s];
      if (tile == kNoTile) {
        if (lane == 0) mbar_arrive(&aggd[s]);
        return;
      }
      const uint32_t epoch = s_epoch;
      const bool fulltile = !(tail_partial && tile == a.ntiles - 1);
      Stage& st = stages[s];
      const unsigned char* tm = tile_mem(s);
      Opt<A> rt[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rt[i] = Opt<A>{A{}, false};
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int ri = (k + int(lane)) & 7;
        const int row = int(lane) * 8 + ri;
        Opt<A> r{A{}, false};
        if (fulltile) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const uint4 v = lds128(tm + swz128(uint32_t(row), uint32_t(c)));
            T x[EPC];
            memcpy(x, &v, 16);
#pragma unroll
            for (int e = 0; e < EPC; ++e) {
              const A y = M::lift(a.f(x[e]));
              r.v = (c == 0 && e == 0) ? y : aop(r.v, y);
            }
          }
          r.has = true;
        } else {
          const uint64_t b = uint64_t(tile) * kTile + uint64_t(row) * IT;
          const uint64_t avail = b < a.n ? a.n - b : 0;
          const int cnt = avail >= uint64_t(IT) ? IT : int(avail);
          for (int q = 0; q < cnt; ++q) {
            const A y = M::lift(a.f(a.src[b + q]));
            r.v = q == 0 ? y : aop(r.v, y);
          }
          r.has = cnt > 0;
        }
        st.rowtot[row] = r;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i == ri) rt[i] = r;
      }
      Opt<A> lt = rt[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) lt = opt_combine(aop, lt, rt[i]);
      lt = warp_reduce_ordered(aop, lt);
      if (lane == 0) {
        const C agg_c = M::to_c(lt.v);
        st.agg = agg_c;
        if (tile == 0) {
          C pre = agg_c;
          if (a.carry_in) pre = cop(M::to_c(M::lift(*a.carry_in)), pre);
          IO::write(a.states, 0, a.state_stride, epoch, kPrefix, pre);
          if (a.ntiles == 1 && a.total_out) *a.total_out = M::CT::to_s(pre);
        } else {
          IO::write(a.states, tile, a.state_stride, epoch, kPartial, agg_c);
        }
        mbar_arrive(&aggd[s]);  // release: row totals + agg visible to the CTA
      }
      __syncwarp();
    }
  }

  if (warp == kWsLookback) {
    constexpr int LB = kWsLookbackPolls;
    constexpr int WIN = kWarp * LB;
    for (uint32_t it = 0;; ++it) {
      const int s = int(it % kWsStages);
      mbar_wait(&aggd[s], (it / kWsStages) & 1u);
      const uint32_t tile = ring[s];
      if (tile == kNoTile) {
        if (lane == 0) mbar_arrive(&carried[s]);  // pass the end marker on to the consumers
        return;
      }
      const uint32_t epoch = s_epoch;
      Stage& st = stages[s];
      Opt<C> carry{C{}, false};
      if (tile == 0) {
        if (a.carry_in) carry = Opt<C>{M::to_c(M::lift(*a.carry_in)), true};
      } else {
        int64_t hi = int64_t(tile);
        for (;;) {
          C val[LB];
          uint32_t kind[LB];
          int first = WIN;
#pragma unroll
          for (int q = 0; q < LB; ++q) {
            kind[q] = 0;
            val[q] = C{};
            const int64_t j = hi - 1 - int64_t(lane) * LB - q;
            if (j >= 0) {
              while ((kind[q] = IO::read(a.states, uint64_t(j), a.state_stride, epoch, val[q])) == 0) {
              }
            }
            if (kind[q] == kPrefix && first == WIN) first = int(lane) * LB + q;
          }
          const unsigned pm = __ballot_sync(kFullMask, first < WIN);
          const int pl = __shfl_sync(kFullMask, first, pm ? __ffs(int(pm)) - 1 : 0);
          const bool found = pm != 0;
          const int lim = found ? pl : WIN - 1;
          Opt<C> v{C{}, false};
#pragma unroll
          for (int q = LB - 1; q >= 0; --q) {
            const int pos = int(lane) * LB + q;
            if (kind[q] != 0 && pos <= lim) v = opt_combine(cop, v, Opt<C>{val[q], true});
          }
#pragma unroll
          for (unsigned d = 1; d < kWarp; d <<= 1) {
            Opt<C> got{shfl_down(v.v, d), __shfl_down_sync(kFullMask, int(v.has), d) != 0};
            if (lane + d < kWarp) v = opt_combine(cop, got, v);
          }
          const Opt<C> window{shfl_idx(v.v, 0), __shfl_sync(kFullMask, int(v.has), 0) != 0};
          carry = opt_combine(cop, window, carry);
          if (found) break;
          hi -= WIN;
        }
        if (lane == 0) {
          const C inclusive_c = cop(carry.v, st.agg);
          IO::write(a.states, tile, a.state_stride, epoch, kPrefix, inclusive_c);
          if (tile == a.ntiles - 1 && a.total_out) *a.total_out = M::CT::to_s(inclusive_c);
        }
      }
      if (lane == 0) {
        st.carry = carry.has ? Opt<A>{M::from_c(carry.v), true} : Opt<A>{A{}, false};
        mbar_arrive(&carried[s]);
      }
      __syncwarp();
    }
  }

  // ---- consumers (warps 0-7)
  for (uint32_t it = 0;; ++it) {
    const int s = int(it % kWsStages);
    mbar_wait(&carried[s], (it / kWsStages) & 1u);
    const uint32_t tile = ring[s];
    if (tile == kNoTile) break;
    Stage& st = stages[s];
    const bool fulltile = !(tail_partial && tile == a.ntiles - 1);
    // block scan of the row totals -> this row's exclusive prefix in the tile
    const Opt<A> tot = st.rowtot[threadIdx.x];
    const Opt<A> incl = warp_scan_incl(aop, tot);
    if (lane == kWarp - 1) s_warp[warp] = incl;
    consumer_sync();
    if (warp == 0) {
      Opt<A> w = lane < NW ? s_warp[lane] : Opt<A>{A{}, false};
      w = warp_scan_incl(aop, w);
      if (lane < NW) s_warp[lane] = w;
    }
    consumer_sync();
    const Opt<A> warp_ex = warp > 0 ? s_warp[warp - 1] : Opt<A>{A{}, false};
    Opt<A> lane_ex = shfl_up_opt(incl, 1);
    if (lane == 0) lane_ex.has = false;
    Opt<A> run = opt_combine(aop, opt_combine(aop, st.carry, warp_ex), lane_ex);
    const uint64_t base = uint64_t(tile) * kTile + uint64_t(threadIdx.x) * IT;
    unsigned char* tm = tile_mem(s);
    if (fulltile) {
      const bool vec = is_aligned(a.dst + base, 16);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint4 v = lds128(tm + swz128(threadIdx.x, c));
        T x[EPC];
        memcpy(x, &v, 16);
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
        S* d = a.dst + base + uint64_t(c) * EPC;
        if (vec) {
          store_items<S, EPC>(d, o);
        } else {
#pragma unroll
          for (int e = 0; e < EPC; ++e) d[e] = o[e];
        }
      }
      if (sizeof(S) == sizeof(T) && tma_store) {
        fence_proxy_async_smem();
        consumer_sync();
        if (threadIdx.x == 0) {
          tma_store_2d(&tmap_out, 0, int(tile) * kScanThreads, tm);
          tma_store_commit();
          tma_store_wait_read();
        }
      } else {
        consumer_sync();
      }
    } else {
      const uint64_t avail = base < a.n ? a.n - base : 0;
      const int cnt = avail >= uint64_t(IT) ? IT : int(avail);
      for (int k = 0; k < cnt; ++k) {
        const A y = M::lift(a.f(a.src[base + k]));
        if constexpr (Inclusive) {
          run.v = run.has ? aop(run.v, y) : y;
          run.has = true;
          a.dst[base + k] = M::lower(run.v);
        } else {
          a.dst[base + k] = run.has ? M::lower(run.v) : a.identity;
          run.v = run.has ? aop(run.v, y) : y;
          run.has = true;
        }
      }
      consumer_sync();
    }
    if (threadIdx.x == 0) mbar_arrive(&empty[s]);
  }
}


}  // namespace forge::cuda
