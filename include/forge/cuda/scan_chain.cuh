// forge/cuda/scan_chain.cuh — persistent scan with a dedicated carry chain.
// Included by forge/cuda/scan.cuh after the shared tile machinery (TileStateIO,
// ScanArgs, ScanMath, TMA helpers); not a standalone header.
#pragma once

namespace forge::cuda {

// ---------------------------------------------------------------------------
// Fast path v6: persistent tiles, aggregates published ahead, one carry chain.
//
// Measured on the one-tile-per-CTA kernel (tools/trace_scan.py):
// a 32 KB tile lives 8.2 us, 5.4 us of it in the decoupled look-back (3.4
// windows of 32 predecessors at ~1.6 us per L2 round trip), and the same kernel
// with the look-back removed streams at 6.1 TB/s.  The look-back is long
// because every tile walks back to the nearest PREFIX on its own, and that
// PREFIX lags the claim frontier by hundreds of tiles.
//
// Here the tile's two halves are split in time instead:
//   reduce(t)  the tile lands in a shared-memory stage (2-D TMA, producer warp);
//              row folds + block scan; the aggregate is published (PARTIAL).
//   chain      ONE warp (in a CTA of its own) walks the tile states in order, 32*Q per
//              L2 round trip: waits for the PARTIALs, scans them, and writes
//              each tile's EXCLUSIVE carry back into its state (PREFIX).
//   fetch      one thread per CTA polls the carries of its tiles in order (with
//              back-off) into their stages' carry slots;
//   scan(t)    D iterations after reduce(t), the workers take the tile's carry
//              — normally already fetched: no look-back at all — and emit the
//              running prefixes from the stage still holding the tile; one TMA
//              tensor store.
// Each CTA owns tiles c, c+G, c+2G, ... (G = grid) and runs, per iteration k,
// reduce(tile k) then scan(tile k-D), with a ring of NS >= D+2 stages so the
// producer keeps NS-D-1 tile loads in flight.  HBM traffic is exactly one read
// and one write of the data; tile states are one 256-byte slot per tile.
//
// Progress: the grid is launched cooperatively (all CTAs co-resident, or the
// launch fails).  A CTA waits only in scan(t), for carry(t), which needs the
// PARTIALs of tiles < t; the owner of such a tile reaches its reduce after
// finishing scans of even smaller tiles only, so by induction on the smallest
// unfinished tile every wait ends.  The chain warp waits only on PARTIALs.

constexpr int kChainWorkers = kScanThreads;               // 8 worker warps
constexpr int kChainProducerWarp = kChainWorkers / kWarp;  // warp 8
constexpr int kChainWarp = kChainProducerWarp + 1;         // warp 9 (chain CTA only)
constexpr int kChainFetchWarp = kChainProducerWarp + 2;    // warp 10
constexpr int kChainThreads = kChainWorkers + 3 * kWarp;   // 352
constexpr int kChainMaxStages = 8;
constexpr int kChainRows = 16;  // chain window: 16 rows x 32 tiles
constexpr uint32_t kPrefixNone = 3;  // carry state "no carry" (tile 0 of a carry-less scan)

__device__ __forceinline__ void worker_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kChainWorkers) : "memory");
}

template <class S, class Op>
struct ChainLayout {
  using A = typename ScanMath<S, Op>::A;
  // per stage: tile bytes + the workers' exclusive in-tile prefixes
  static constexpr uint32_t kExBytes = uint32_t((sizeof(Opt<A>) * kChainWorkers + 1023) / 1024 * 1024);
  static constexpr uint32_t kStageBytes = kSmemTileBytes + kExBytes;
  static uint32_t dyn_bytes(int ns) { return uint32_t(ns) * kStageBytes + 1024; }
};

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kChainThreads, 1)
    scan_chain_kernel(const ScanArgs<T, S, F, Op> a, const __grid_constant__ CUtensorMap tmap,
                      const __grid_constant__ CUtensorMap tmap_out, bool tma_store, int ns, int lag) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  using L = ChainLayout<S, Op>;
  constexpr int IT = smem_scan_items<T>();
  constexpr int EPC = 16 / int(sizeof(T));
  constexpr int NCH = kRowBytes / 16;
  constexpr int NW = kChainWorkers / kWarp;
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t full[kChainMaxStages], empty[kChainMaxStages], carried[kChainMaxStages];
  __shared__ uint32_t s_epoch;
  __shared__ Opt<A> s_warp[NW];
  __shared__ Opt<A> s_carry[kChainMaxStages];
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };
  unsigned char* base_mem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  auto stage_tile = [&](int s) { return base_mem + size_t(s) * L::kStageBytes; };
  auto stage_carry = [&](int s) { return &s_carry[s]; };
  auto stage_ex = [&](int s) {
    return reinterpret_cast<Opt<A>*>(base_mem + size_t(s) * L::kStageBytes + kSmemTileBytes);
  };
  const unsigned warp = threadIdx.x / kWarp, lane = lane_id();
  // The LAST CTA runs only the carry chain (an SM of its own: measured, the
  // chain warp is latency-bound and slows down next to busy workers).
  const uint32_t G = gridDim.x - 1, c = blockIdx.x;
  const bool chain_cta = c == G;
  const uint32_t my_tiles = !chain_cta && c < a.ntiles ? (a.ntiles - 1 - c) / G + 1 : 0;
  auto tile_of = [&](uint32_t k) { return c + k * G; };
  auto full_tile = [&](uint32_t t) { return uint64_t(t + 1) * kTile <= a.n; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&carried[s], 1);
    }
    fence_mbar_init();
    // epoch, then one acq_rel arrival per CTA; the last arrival advances the
    // epoch for the next launch (stale states then read as INVALID).
    const uint32_t e = ld_acquire_gpu(a.ctrl + 2);
    const uint32_t t = atom_add_acq_rel_gpu(a.ctrl + 0, 1u);
    if (t == gridDim.x - 1) {
      st_relaxed_gpu(a.ctrl + 0, 0u);
      st_relaxed_gpu(a.ctrl + 2, e + 1u);
    }
    s_epoch = e;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;

  if (warp == kChainProducerWarp) {
    // ---- producer: 2-D TMA of each owned tile into the ring
    if (lane != 0) return;
    for (uint32_t k = 0; k < my_tiles; ++k) {
      const int s = int(k % uint32_t(ns));
      if (k >= uint32_t(ns)) mbar_wait(&empty[s], ((k / uint32_t(ns)) - 1) & 1u);
      const uint32_t t = tile_of(k);
      if (a.trace) a.trace[uint64_t(t) * 8 + 0] = global_ns();
      if (full_tile(t)) {
        mbar_arrive_expect_tx(&full[s], kSmemTileBytes);
        tma_load_2d(stage_tile(s), &tmap, 0, int(t) * kScanThreads, &full[s]);
      } else {
        mbar_arrive(&full[s]);  // partial last tile: the workers read it from global
      }
    }
    return;
  }

  if (warp == kChainWarp) {
    // ---- carry chain (last CTA): exclusive carry of every tile, in order.
    // Sliding window of kChainRows rows x 32 tiles (tile base + 32q + lane in
    // row q): every round polls the window's missing PARTIALs (all loads in
    // flight together), then retires every complete row at the front — each
    // row one ordered warp scan — and slides.  The chain trails the PARTIAL
    // frontier by about one L2 round trip, whatever the window size.
    if (!chain_cta) return;
    Opt<C> carry{C{}, false};
    if (a.carry_in) carry = Opt<C>{M::to_c(M::lift(*a.carry_in)), true};
    C val[kChainRows];
    bool ok[kChainRows];
#pragma unroll
    for (int q = 0; q < kChainRows; ++q) ok[q] = false;
    uint64_t base = 0;
    uint32_t rounds = 0;
    uint64_t* rtrace = a.trace ? a.trace + uint64_t(a.ntiles) * 8 : nullptr;
    while (base < a.ntiles) {
      ++rounds;
      if (rtrace && lane == 0 && rounds < 2048) rtrace[rounds * 4 + 0] = global_ns();
      {
        uint64_t raw[kChainRows][IO::STRIDE];
#pragma unroll
        for (int q = 0; q < kChainRows; ++q) {
          const uint64_t j = base + uint64_t(q) * kWarp + lane;
          if (!ok[q] && j < a.ntiles) IO::load_raw(a.states, j, a.state_stride, raw[q]);
        }
#pragma unroll
        for (int q = 0; q < kChainRows; ++q) {
          const uint64_t j = base + uint64_t(q) * kWarp + lane;
          if (!ok[q]) ok[q] = j >= a.ntiles || IO::decode(raw[q], epoch, val[q]) == kPartial;
        }
      }
      int nready = 0;
#pragma unroll
      for (int q = 0; q < kChainRows; ++q)
        if (nready == q && __all_sync(kFullMask, ok[q])) nready = q + 1;
      if (rtrace && lane == 0 && rounds < 2048) {
        rtrace[rounds * 4 + 1] = global_ns();
        rtrace[rounds * 4 + 3] = nready;
      }
      // row scans are independent (interleaved); only the carry is serial
      Opt<C> li[kChainRows];
#pragma unroll
      for (int q = 0; q < kChainRows; ++q) {
        const uint64_t j = base + uint64_t(q) * kWarp + lane;
        li[q] = Opt<C>{val[q], q < nready && j < a.ntiles};
        if (q < nready) li[q] = warp_scan_incl(cop, li[q]);
      }
#pragma unroll
      for (int q = 0; q < kChainRows; ++q) {
        if (q < nready) {
          const uint64_t j = base + uint64_t(q) * kWarp + lane;
          Opt<C> lex = shfl_up_opt(li[q], 1);
          if (lane == 0) lex.has = false;
          const Opt<C> tot = shfl_idx_opt(li[q], kWarp - 1);
          const Opt<C> ex = opt_combine(cop, carry, lex);
          if (j < a.ntiles) IO::write(a.states, j, a.state_stride, epoch, ex.has ? kPrefix : kPrefixNone, ex.v);
          if (a.trace && j < a.ntiles) {
            a.trace[j * 8 + 2] = global_ns();
            a.trace[j * 8 + 7] = (uint64_t(rounds) << 8) | uint64_t(nready);
          }
          carry = opt_combine(cop, carry, tot);
        }
      }
      // slide the window by nready rows (warp-uniform)
#pragma unroll
      for (int r = 0; r < kChainRows; ++r) {
        if (r < nready) {
#pragma unroll
          for (int q = 0; q + 1 < kChainRows; ++q) {
            val[q] = val[q + 1];
            ok[q] = ok[q + 1];
          }
          ok[kChainRows - 1] = false;
        }
      }
      base += uint64_t(nready) * kWarp;
      if (rtrace && lane == 0 && rounds < 2048) rtrace[rounds * 4 + 2] = global_ns();
    }
    if (lane == 0 && a.total_out) *a.total_out = M::CT::to_s(carry.v);
    return;
  }

  if (warp == kChainFetchWarp) {
    // ---- carry fetcher: one lane fetches the carries of the CTA's tiles in
    // order, each once its stage holds the tile (the previous occupant has
    // then consumed its carry), into the stage's slot.  Polls back off: the
    // tile-state lines are shared with the chain, and 148 CTAs spinning on
    // them would slow the chain down (measured).
    if (lane != 0) return;
    for (uint32_t k = 0; k < my_tiles; ++k) {
      const int s = int(k % uint32_t(ns));
      mbar_wait(&full[s], (k / uint32_t(ns)) & 1u);
      C cv{};
      uint32_t kind;
      while ((kind = IO::read(a.states, tile_of(k), a.state_stride, epoch, cv)) < kPrefix) __nanosleep(256);
      *stage_carry(s) = Opt<A>{kind == kPrefix ? M::from_c(cv) : A{}, kind == kPrefix};
      if (a.trace) a.trace[uint64_t(tile_of(k)) * 8 + 3] = global_ns();
      mbar_arrive(&carried[s]);
    }
    return;
  }

  // ---- workers
  for (uint32_t k = 0; k < my_tiles + uint32_t(lag); ++k) {
    if (k < my_tiles) {
      // reduce(tile k): row folds, block scan -> exclusive in-tile prefixes, PARTIAL
      const int s = int(k % uint32_t(ns));
      const uint32_t t = tile_of(k);
      const bool fullt = full_tile(t);
      const uint64_t base = uint64_t(t) * kTile + uint64_t(threadIdx.x) * IT;
      mbar_wait(&full[s], (k / uint32_t(ns)) & 1u);
      Opt<A> tot{A{}, false};
      if (fullt) {
        const unsigned char* tm = stage_tile(s);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const uint4 v = lds128(tm + swz128(threadIdx.x, ch));
          T x[EPC];
          memcpy(x, &v, 16);
#pragma unroll
          for (int e = 0; e < EPC; ++e) {
            const A y = M::lift(a.f(x[e]));
            tot.v = (ch == 0 && e == 0) ? y : aop(tot.v, y);
          }
        }
        tot.has = true;
      } else {
        const uint64_t avail = base < a.n ? a.n - base : 0;
        const int cnt = avail >= uint64_t(IT) ? IT : int(avail);
        for (int i = 0; i < cnt; ++i) {
          const A y = M::lift(a.f(a.src[base + i]));
          tot.v = i == 0 ? y : aop(tot.v, y);
        }
        tot.has = cnt > 0;
      }
      const Opt<A> incl = warp_scan_incl(aop, tot);
      if (lane == kWarp - 1) s_warp[warp] = incl;
      worker_sync();
      if (warp == 0) {
        Opt<A> w = lane < NW ? s_warp[lane] : Opt<A>{A{}, false};
        w = warp_scan_incl(aop, w);
        if (lane < NW) s_warp[lane] = w;
      }
      worker_sync();
      const Opt<A> warp_ex = warp > 0 ? s_warp[warp - 1] : Opt<A>{A{}, false};
      Opt<A> lane_ex = shfl_up_opt(incl, 1);
      if (lane == 0) lane_ex.has = false;
      stage_ex(s)[threadIdx.x] = opt_combine(aop, warp_ex, lane_ex);
      if (threadIdx.x == 0) {
        const Opt<A> agg = s_warp[NW - 1];  // every tile holds >= 1 element
        IO::write(a.states, t, a.state_stride, epoch, kPartial, M::to_c(agg.v));
        if (a.trace) {
          a.trace[uint64_t(t) * 8 + 1] = global_ns();
          a.trace[uint64_t(t) * 8 + 6] = c;
        }
      }
      worker_sync();  // s_warp is reused
    }
    if (k >= uint32_t(lag)) {
      // scan(tile k - lag): carry from the chain, running prefixes, TMA store
      const uint32_t kk = k - uint32_t(lag);
      const int s = int(kk % uint32_t(ns));
      const uint32_t t = tile_of(kk);
      const bool fullt = full_tile(t);
      const uint64_t base = uint64_t(t) * kTile + uint64_t(threadIdx.x) * IT;
      mbar_wait(&carried[s], (kk / uint32_t(ns)) & 1u);
      if (a.trace && threadIdx.x == 0) a.trace[uint64_t(t) * 8 + 4] = global_ns();
      Opt<A> run = opt_combine(aop, *stage_carry(s), stage_ex(s)[threadIdx.x]);
      unsigned char* tm = stage_tile(s);
      if (fullt) {
        const bool vec = is_aligned(a.dst + base, 16);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const uint4 v = lds128(tm + swz128(threadIdx.x, ch));
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
              asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(tm + swz128(threadIdx.x, ch))),
                           "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                           : "memory");
              continue;
            }
          }
          S* d = a.dst + base + uint64_t(ch) * EPC;
          if (vec) {
            store_items<S, EPC>(d, o);
          } else {
#pragma unroll
            for (int e = 0; e < EPC; ++e) d[e] = o[e];
          }
        }
        if (sizeof(S) == sizeof(T) && tma_store) {
          fence_proxy_async_smem();
          worker_sync();
          if (threadIdx.x == 0) {
            tma_store_2d(&tmap_out, 0, int(t) * kScanThreads, tm);
            tma_store_commit();
            tma_store_wait_read();
          }
        } else {
          worker_sync();
        }
      } else {
        const uint64_t avail = base < a.n ? a.n - base : 0;
        const int cnt = avail >= uint64_t(IT) ? IT : int(avail);
        for (int i = 0; i < cnt; ++i) {
          const A y = M::lift(a.f(a.src[base + i]));
          if constexpr (Inclusive) {
            run.v = run.has ? aop(run.v, y) : y;
            run.has = true;
            a.dst[base + i] = M::lower(run.v);
          } else {
            a.dst[base + i] = run.has ? M::lower(run.v) : a.identity;
            run.v = run.has ? aop(run.v, y) : y;
            run.has = true;
          }
        }
        worker_sync();
      }
      if (threadIdx.x == 0) mbar_arrive(&empty[s]);  // stage free for the producer
      if (a.trace && threadIdx.x == 0) a.trace[uint64_t(t) * 8 + 5] = global_ns();
    }
  }
  if (threadIdx.x == 0) tma_store_wait_read();
}

}  // namespace forge::cuda
