// forge/cuda/scan_cluster.cuh — cluster-tiled decoupled look-back scan.
// Included by forge/cuda/scan.cuh after the shared tile machinery (TileStateIO,
// ScanArgs, ScanMath, TMA helpers); not a standalone header.
#pragma once

namespace forge::cuda {

// ---------------------------------------------------------------------------
// Fast path v5: one look-back tile per thread-block CLUSTER.
//
// Why: with one 32 KB tile per CTA, ~900 tiles are in flight and tickets are
// claimed at ~100 tiles/us at the bandwidth target; a tile's nearest PREFIX is
// then (look-back duration x claim rate) tiles back, several 32-tile windows —
// each one an L2 round trip — so the look-back grows with the lag it causes
// (measured: 5.4 us of an 8 us tile lifetime).  The lag is set by
// the number of TILE STATES per byte, not by the bytes: a cluster of K CTAs
// (K x 32 KB, K SMs of one GPC) publishes ONE state, so the claim rate and the
// lag drop K-fold and the look-back usually ends in the first window.
//
// Per cluster tile t (claimed by rank 0's ticket, broadcast over DSMEM):
//   every CTA   2-D TMA of its 32 KB sub-tile t*K + rank; pass 1 folds rows;
//               block scan; its aggregate -> the leader's smem (st.shared::cluster)
//               + remote mbarrier arrive (release.cluster);
//   leader w0   ordered fold of the K aggregates -> PARTIAL; look-back over
//               cluster-tile states -> PREFIX; each CTA's carry (carry ⊕ aggs of
//               lower ranks) -> that CTA's smem + remote arrive;
//   every CTA   pass 2: running prefixes written back into the tile, one TMA
//               tensor store.
// Progress: clusters are co-scheduled (all K CTAs resident together); tickets
// are claimed in order and a leader waits only on smaller tickets' states.
// A CTA touches a peer's shared memory only while that peer is blocked on a
// barrier the access itself completes, so no CTA exits under a remote access.

constexpr int kMaxScanCluster = 8;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// Address of the same shared variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// Copies a value word by word into CTA `rank`'s copy of `*local`.
template <class V>
__device__ __forceinline__ void st_cluster_value(V* local, uint32_t rank, const V& v) {
  static_assert(sizeof(V) % 4 == 0, "cluster stores move 32-bit words");
  const uint32_t base = mapa_shared(local, rank);
  uint32_t w[sizeof(V) / 4];
  memcpy(w, &v, sizeof(V));
#pragma unroll
  for (int i = 0; i < int(sizeof(V) / 4); ++i) st_cluster_u32(base + 4u * i, w[i]);
}

// A carry value plus its validity flag as a whole 32-bit word (Opt<C> may
// pack the flag into padding; DSMEM stores here move 32-bit words).
template <class C>
struct ClusterCarryW {
  C v;
  uint32_t has;
};

template <class A, class C>
struct ClusterShared {
  Opt<A> warp[kScanThreads / kWarp];
  uint32_t tile, epoch;                 // written by the leader
  ClusterCarryW<C> aggs[kMaxScanCluster];  // leader only: sub-tile aggregates, by rank
  ClusterCarryW<C> carry;               // written by the leader: carry into this sub-tile
};

template <class S, class Op>
using ClusterSharedOf = ClusterShared<typename ScanMath<S, Op>::A, typename ScanMath<S, Op>::C>;

template <class T, class S, class F, class Op, bool Inclusive>
__global__ void __launch_bounds__(kScanThreads)
    scan_cluster_kernel(const ScanArgs<T, S, F, Op> a, const __grid_constant__ CUtensorMap tmap,
                        const __grid_constant__ CUtensorMap tmap_out, bool tma_store) {
  using M = ScanMath<S, Op>;
  using A = typename M::A;
  using C = typename M::C;
  using IO = TileStateIO<C>;
  static_assert(sizeof(ClusterCarryW<C>) % 4 == 0, "carry slots move as 32-bit words");
  constexpr int IT = smem_scan_items<T>();
  constexpr int EPC = 16 / int(sizeof(T));
  constexpr int NCH = kRowBytes / 16;
  constexpr int NW = kScanThreads / kWarp;
  constexpr uint64_t kTile = uint64_t(kScanThreads) * IT;
  extern __shared__ unsigned char dyn_smem[];
  __shared__ __align__(8) uint64_t bar_tma, bar_tk, bar_agg, bar_carry;
  __shared__ uint32_t s_phase;
  __shared__ ClusterSharedOf<S, Op> sh;
  auto aop = [&](const A& x, const A& y) { return M::comb(a.op, x, y); };
  auto cop = [&](const C& x, const C& y) { return M::CT::op(a.op, x, y); };
  unsigned char* tile_mem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn_smem) + 1023) & ~uintptr_t(1023));
  const uint32_t rank = cluster_ctarank(), K = cluster_nctarank();
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;

  // ---- setup: barriers, speculative TMA of sub-tile clusterid*K + rank, ticket
  const uint32_t g = cluster_id_x() * K + rank;
  const bool gfull = uint64_t(g + 1) * kTile <= a.n;
  uint32_t t_claim = 0, e_claim = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_tk, 1);
    mbar_init(&bar_agg, K);
    mbar_init(&bar_carry, 1);
    fence_mbar_init();
    if (gfull) {
      mbar_arrive_expect_tx(&bar_tma, kSmemTileBytes);
      tma_load_2d(tile_mem, &tmap, 0, int(g) * kScanThreads, &bar_tma);
    }
  }
  cluster_arrive_relaxed();  // (release of the mbarrier inits is fence_mbar_init's)
  if (rank == 0 && threadIdx.x == 0) {
    e_claim = ld_acquire_gpu(a.ctrl + 2);
    t_claim = atom_add_acq_rel_gpu(a.ctrl + 0, 1u);
    if (t_claim == a.ntiles - 1) {
      st_relaxed_gpu(a.ctrl + 0, 0u);
      st_relaxed_gpu(a.ctrl + 2, e_claim + 1u);
    }
  }
  cluster_wait();  // every CTA of the cluster has started and initialised its barriers
  if (rank == 0 && threadIdx.x < K) {
    const uint32_t r = threadIdx.x;
    const uint32_t t = __shfl_sync(__activemask(), t_claim, 0), e = __shfl_sync(__activemask(), e_claim, 0);
    st_cluster_u32(mapa_shared(&sh.tile, r), t);
    st_cluster_u32(mapa_shared(&sh.epoch, r), e);
    mbar_arrive_cluster(mapa_shared(&bar_tk, r));
  }
  if (threadIdx.x == 0) {
    mbar_wait_cluster(&bar_tk, 0);
    const uint32_t sub = sh.tile * K + rank;
    s_phase = 0;
    if (sub != g) {
      if (gfull) mbar_wait(&bar_tma, 0);  // drain the speculative copy
      if (uint64_t(sub + 1) * kTile <= a.n) {
        mbar_arrive_expect_tx(&bar_tma, kSmemTileBytes);
        tma_load_2d(tile_mem, &tmap, 0, int(sub) * kScanThreads, &bar_tma);
        s_phase = gfull ? 1u : 0u;
      }
    }
  }
  __syncthreads();
  const uint32_t ctile = sh.tile, epoch = sh.epoch;
  const uint64_t sub = uint64_t(ctile) * K + rank;
  const bool full = (sub + 1) * kTile <= a.n;
  const uint64_t base = sub * kTile + uint64_t(threadIdx.x) * IT;
  const uint64_t avail = base < a.n ? a.n - base : 0;
  const int count = full ? IT : (avail >= uint64_t(IT) ? IT : int(avail));
  trace_mark(a.trace, sub, 0);
  if (a.trace && threadIdx.x == 0) {
    uint32_t sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    a.trace[sub * 8 + 5] = sm;
  }

  // ---- pass 1: ordered fold of this thread's row
  Opt<A> tot{A{}, false};
  if (full) {
    mbar_wait(&bar_tma, s_phase);
    trace_mark(a.trace, sub, 1);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 v = lds128(tile_mem + swz128(threadIdx.x, c));
      T x[EPC];
      memcpy(x, &v, 16);
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const A y = M::lift(a.f(x[e]));
        tot.v = (c == 0 && e == 0) ? y : aop(tot.v, y);
      }
    }
    tot.has = true;
  } else {
    for (int k = 0; k < count; ++k) {
      const A y = M::lift(a.f(a.src[base + k]));
      tot.v = k == 0 ? y : aop(tot.v, y);
    }
    tot.has = count > 0;
  }

  // ---- block scan of the row totals
  const Opt<A> incl = warp_scan_incl(aop, tot);
  if (lane == kWarp - 1) sh.warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    Opt<A> w = lane < NW ? sh.warp[lane] : Opt<A>{A{}, false};
    w = warp_scan_incl(aop, w);
    if (lane < NW) sh.warp[lane] = w;
  }
  __syncthreads();

  // ---- sub-tile aggregate -> leader
  if (threadIdx.x == 0) {
    const Opt<A> agg = sh.warp[NW - 1];
    ClusterCarryW<C> w;
    w.v = agg.has ? M::to_c(agg.v) : C{};
    w.has = agg.has ? 1u : 0u;
    st_cluster_value(&sh.aggs[rank], 0, w);
    mbar_arrive_cluster(mapa_shared(&bar_agg, 0));
  }
  trace_mark(a.trace, sub, 2);

  // ---- leader: cluster-tile aggregate, publication, look-back, carries out
  if (rank == 0 && warp == 0) {
    mbar_wait_cluster(&bar_agg, 0);
    // lane r < K: aggregate of sub-tile r; ordered inclusive scan over ranks.
    Opt<C> ar{C{}, false};
    if (lane < K) ar = Opt<C>{sh.aggs[lane].v, sh.aggs[lane].has != 0};
    const Opt<C> ar_incl = warp_scan_incl(cop, ar);
    const Opt<C> cagg = shfl_idx_opt(ar_incl, int(K) - 1);  // >= 1 element: sub-tile 0 is non-empty
    Opt<C> carry{C{}, false};
    if (ctile == 0) {
      if (a.carry_in) carry = Opt<C>{M::to_c(M::lift(*a.carry_in)), true};
      if (lane == 0) {
        const C pre = carry.has ? cop(carry.v, cagg.v) : cagg.v;
        IO::write(a.states, 0, a.state_stride, epoch, kPrefix, pre);
        if (a.ntiles == 1 && a.total_out) *a.total_out = M::CT::to_s(pre);
      }
    } else {
      if (lane == 0) IO::write(a.states, ctile, a.state_stride, epoch, kPartial, cagg.v);
      int64_t hi = int64_t(ctile);
      uint32_t windows = 0;
      for (;;) {
        ++windows;
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
      if (a.trace && lane == 0) a.trace[sub * 8 + 6] = windows;
      if (lane == 0) {
        const C inclusive_c = cop(carry.v, cagg.v);
        IO::write(a.states, ctile, a.state_stride, epoch, kPrefix, inclusive_c);
        if (ctile == a.ntiles - 1 && a.total_out) *a.total_out = M::CT::to_s(inclusive_c);
      }
    }
    // carry into sub-tile r = carry ⊕ aggs[0..r-1]
    Opt<C> ar_ex = shfl_up_opt(ar_incl, 1);
    if (lane == 0) ar_ex.has = false;
    const Opt<C> cr = opt_combine(cop, carry, ar_ex);
    if (lane < K) {
      ClusterCarryW<C> w;
      w.v = cr.v;
      w.has = cr.has ? 1u : 0u;
      st_cluster_value(&sh.carry, lane, w);
      mbar_arrive_cluster(mapa_shared(&bar_carry, lane));
    }
  }
  if (threadIdx.x == 0) mbar_wait_cluster(&bar_carry, 0);
  __syncthreads();
  trace_mark(a.trace, sub, 3);
  if (count == 0) return;

  const Opt<A> tile_ex{sh.carry.has ? M::from_c(sh.carry.v) : A{}, sh.carry.has != 0};
  const Opt<A> warp_ex = warp > 0 ? sh.warp[warp - 1] : Opt<A>{A{}, false};
  Opt<A> lane_ex = shfl_up_opt(incl, 1);
  if (lane == 0) lane_ex.has = false;
  Opt<A> run = opt_combine(aop, opt_combine(aop, tile_ex, warp_ex), lane_ex);

  // ---- pass 2: running prefixes
  if (full) {
    const bool vec = is_aligned(a.dst + base, 16);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 v = lds128(tile_mem + swz128(threadIdx.x, c));
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
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_addr(tile_mem + swz128(threadIdx.x, c))),
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
      __syncthreads();
      if (threadIdx.x == 0) {
        tma_store_2d(&tmap_out, 0, int(sub) * kScanThreads, tile_mem);
        tma_store_commit();
        tma_store_wait_read();
      }
    }
    trace_mark(a.trace, sub, 4);
  } else {
    for (int k = 0; k < count; ++k) {
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
  }
}

}  // namespace forge::cuda
