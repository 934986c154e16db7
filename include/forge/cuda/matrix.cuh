// forge/cuda/matrix.cuh — semiring matrix-vector kernels for sm_100a.
//
// Reference: prim::matvec / prim::vecmat and detail_mat::{tall,wide}_kernel,
// run_mat, plan_mat (primitives.hpp:204-244, 611-807).  A is n x p column-major
// (element (i,j) at j*n + i).
//
//   matvec (BLAS gemv 'T', "gevm")   y[j] = op_i f(x[i], A[i,j])
//     The fold runs down a CONTIGUOUS column.  One warp per (column, row-split);
//     lanes read 256-bit vectors of the column (ld.global.nc.L1::no_allocate)
//     and of x (cached: x is re-read by every column and stays in L1/L2).
//     Commutative ops: lanes stride the column (coalesced) and reduce with a
//     butterfly.  Non-commutative ops: lane L owns a contiguous run of rows and
//     the warp reduces in lane order (the reference's tall path keeps row order
//     the same way, primitives.hpp:606-610).  Tall-skinny shapes split the rows
//     across warps; the last split to finish (ticket per column) folds the
//     split partials in split order.
//
//   vecmat (BLAS gemv 'N', "gemv")   z[i] = op_j f(A[i,j], x[j])
//     The fold runs ACROSS columns, so the reference's per-output row view is
//     strided (primitives.hpp:793-807).  Here every thread owns VE consecutive
//     rows and walks its columns in order: each step is one 256-bit coalesced
//     load of A[i..i+VE, j] plus a warp-uniform x[j].  Columns are split across
//     blocks; the last block of a row-block (ticket) folds the split partials in
//     split order.  Column order is preserved everywhere, so any associative op
//     is valid.
//
// No tensor cores: both are HBM-bound streaming kernels (<= 0.5 flop/byte).
#pragma once

#include "forge/cuda/reduce.cuh"

namespace forge::cuda {

constexpr int kMatThreads = 256;
constexpr int kMatWarps = kMatThreads / kWarp;

template <class T, class S, class F2, class Op>
struct GevmArgs {
  const T* A;
  const T* x;  // nullable when !UsesX
  S* y;
  uint64_t n, p;
  uint64_t lda;  // elements between columns (>= n): a block of a larger column-major matrix
  F2 f;        // f(x_elem, a_elem)
  Op op;
  uint32_t ks;              // row splits per column
  uint64_t rows_per_split;  // multiple of 32 * VE
  bool vec;                 // 256-bit path allowed (alignment)
  S* partials;              // [p][ks]
  uint32_t* tickets;        // [p]
};

template <class T, class S, class F2, class Op, bool UsesX, bool Ordered>
__global__ void __launch_bounds__(kMatThreads) gevm_kernel(const GevmArgs<T, S, F2, Op> a) {
  constexpr int VE = mr_vec_elems<T>();
  constexpr int U = 4;
  __shared__ bool s_last[kMatWarps];
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  const uint64_t item = uint64_t(blockIdx.x) * kMatWarps + warp;
  if (item >= a.p * a.ks) return;
  const uint64_t j = item / a.ks;
  const uint32_t s = uint32_t(item % a.ks);
  const uint64_t r0 = uint64_t(s) * a.rows_per_split;
  const uint64_t r1 = r0 + a.rows_per_split < a.n ? r0 + a.rows_per_split : a.n;
  const T* col = a.A + j * a.lda;
  const T xz{};
  auto fx = [&](const T& xv, const T& av) { return a.f(UsesX ? xv : xz, av); };

  Opt<S> acc{S{}, false};
  if constexpr (!Ordered) {
    if (a.vec && VE > 1) {
      const uint64_t nv = (r1 - r0) / VE;  // r0 is a multiple of 32*VE
      const T* cv = col + r0;
      const T* xv = a.x ? a.x + r0 : nullptr;
      uint64_t k = lane;
      S vacc[VE];
      bool vh = false;
      for (; k + uint64_t(kWarp) * (U - 1) < nv; k += uint64_t(kWarp) * U) {
        T av[U][VE], xx[U][VE];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          load_items<T, VE>(cv + (k + u * kWarp) * VE, av[u]);
          if constexpr (UsesX) load_items<T, VE, false>(xv + (k + u * kWarp) * VE, xx[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < VE; ++e) {
            S t = fx(UsesX ? xx[u][e] : xz, av[u][e]);
            vacc[e] = (vh || u > 0) ? a.op(vacc[e], t) : t;
          }
        vh = true;
      }
      for (; k < nv; k += kWarp) {
        T av[VE], xx[VE];
        load_items<T, VE>(cv + k * VE, av);
        if constexpr (UsesX) load_items<T, VE, false>(xv + k * VE, xx);
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          S t = fx(UsesX ? xx[e] : xz, av[e]);
          vacc[e] = vh ? a.op(vacc[e], t) : t;
        }
        vh = true;
      }
      if (vh) {
        S t = vacc[0];
#pragma unroll
        for (int e = 1; e < VE; ++e) t = a.op(t, vacc[e]);
        acc = Opt<S>{t, true};
      }
      for (uint64_t i = r0 + nv * VE + lane; i < r1; i += kWarp)
        acc = opt_combine(a.op, acc, Opt<S>{fx(UsesX ? a.x[i] : xz, col[i]), true});
    } else {
      for (uint64_t i = r0 + lane; i < r1; i += kWarp)
        acc = opt_combine(a.op, acc, Opt<S>{fx(UsesX ? a.x[i] : xz, col[i]), true});
    }
    acc = warp_allreduce_comm(a.op, acc);
  } else {
    // Lane-contiguous runs of rows, folded in row order, then an ordered warp tree.
    const uint64_t len = r1 - r0;
    uint64_t per = ceil_div(len, kWarp);
    if (VE > 1) per = round_up(per, VE);
    const uint64_t lo = r0 + lane * per < r1 ? r0 + lane * per : r1;
    const uint64_t hi = lo + per < r1 ? lo + per : r1;
    uint64_t i = lo;
    if (a.vec && VE > 1) {
      for (; i + VE <= hi; i += VE) {
        T av[VE], xx[VE];
        load_items<T, VE>(col + i, av);
        if constexpr (UsesX) load_items<T, VE, false>(a.x + i, xx);
#pragma unroll
        for (int e = 0; e < VE; ++e)
          acc = opt_combine(a.op, acc, Opt<S>{fx(UsesX ? xx[e] : xz, av[e]), true});
      }
    }
    for (; i < hi; ++i) acc = opt_combine(a.op, acc, Opt<S>{fx(UsesX ? a.x[i] : xz, col[i]), true});
    acc = warp_reduce_ordered(a.op, acc);
  }

  if (a.ks == 1) {
    if (lane == 0) a.y[j] = acc.v;
    return;
  }
  // Split partial; the last split to arrive folds all splits in order.
  if (lane == 0) {
    a.partials[j * a.ks + s] = acc.v;
    const uint32_t t = atom_add_acq_rel_gpu(a.tickets + j, 1u);
    s_last[warp] = (t == a.ks - 1);
    if (s_last[warp]) st_relaxed_gpu(a.tickets + j, 0u);
  }
  __syncwarp();
  if (!s_last[warp]) return;
  if (lane == 0) {
    S v = ld_strong(a.partials + j * a.ks);
    for (uint32_t q = 1; q < a.ks; ++q) v = a.op(v, ld_strong(a.partials + j * a.ks + q));
    a.y[j] = v;
  }
}

// Column-group variant for commutative ops on aligned data (the common case):
// a warp owns CPW adjacent columns and a row split; every step a lane loads
// its 32 bytes of x ONCE and 32 bytes of each of the CPW columns, so x costs
// one load per CPW columns and the registers a warp keeps in flight are almost
// all A (the one-column kernel holds as much x as A in flight, 100 registers,
// 2 CTAs/SM).  Split partials are folded in split order by the last split of
// the group (ticket of its first column).
template <class T, class S, class F2, class Op, bool UsesX, int CPW, int MINB = 1>
__global__ void __launch_bounds__(kMatThreads, MINB) gevm_cols_kernel(const GevmArgs<T, S, F2, Op> a) {
  constexpr int VE = mr_vec_elems<T>();
  __shared__ bool s_last[kMatWarps];
  const unsigned lane = lane_id(), warp = threadIdx.x / kWarp;
  const uint64_t groups = ceil_div(a.p, CPW);
  const uint64_t item = uint64_t(blockIdx.x) * kMatWarps + warp;
  if (item >= groups * a.ks) return;
  const uint64_t grp = item / a.ks;
  const uint32_t s = uint32_t(item % a.ks);
  const uint64_t j0 = grp * CPW;
  const int nc = a.p - j0 < uint64_t(CPW) ? int(a.p - j0) : CPW;
  const uint64_t r0 = uint64_t(s) * a.rows_per_split;
  const uint64_t r1 = r0 + a.rows_per_split < a.n ? r0 + a.rows_per_split : a.n;
  const T xz{};
  auto fx = [&](const T& xv, const T& av) { return a.f(UsesX ? xv : xz, av); };

  S acc[CPW];
  bool has = false;
  const uint64_t nv = (r1 - r0) / VE;  // r0 is a multiple of 32 * VE
  for (uint64_t k = lane; k < nv; k += kWarp) {
    const uint64_t i = r0 + k * VE;
    T xx[VE], av[CPW][VE];
    if constexpr (UsesX) load_items<T, VE, false>(a.x + i, xx);
#pragma unroll
    for (int c = 0; c < CPW; ++c)
      if (c < nc) load_items<T, VE>(a.A + (j0 + c) * a.lda + i, av[c]);
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const S t = fx(UsesX ? xx[e] : xz, av[c][e]);
        acc[c] = (has || e > 0) ? a.op(acc[c], t) : t;
      }
    }
    has = true;
  }
  Opt<S> part[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) part[c] = Opt<S>{acc[c], has};
  for (uint64_t i = r0 + nv * VE + lane; i < r1; i += kWarp) {
#pragma unroll
    for (int c = 0; c < CPW; ++c)
      if (c < nc) part[c] = opt_combine(a.op, part[c], Opt<S>{fx(UsesX ? a.x[i] : xz, a.A[(j0 + c) * a.lda + i]), true});
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c) part[c] = warp_allreduce_comm(a.op, part[c]);

  if (a.ks == 1) {
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < CPW; ++c)
        if (c < nc) a.y[j0 + c] = part[c].v;
    }
    return;
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < CPW; ++c)
      if (c < nc) a.partials[(j0 + c) * a.ks + s] = part[c].v;
    const uint32_t t = atom_add_acq_rel_gpu(a.tickets + j0, 1u);
    s_last[warp] = (t == a.ks - 1);
    if (s_last[warp]) st_relaxed_gpu(a.tickets + j0, 0u);
  }
  __syncwarp();
  if (!s_last[warp]) return;
  // lane c < nc folds column j0 + c in split order
  if (int(lane) < nc) {
    const S* pp = a.partials + (j0 + lane) * a.ks;
    S v = ld_strong(pp);
    for (uint32_t q = 1; q < a.ks; ++q) v = a.op(v, ld_strong(pp + q));
    a.y[j0 + lane] = v;
  }
}

template <class T, class S, class F2, class Op>
struct GemvArgs {
  const T* A;
  const T* x;
  S* z;
  uint64_t n, p;
  uint64_t lda;  // elements between columns (>= n): a row block of a larger matrix, in place
  F2 f;  // f(a_elem, x_elem)
  Op op;
  uint32_t ks;              // column splits
  uint64_t cols_per_split;
  uint32_t row_blocks;
  bool vec;
  S* partials;        // [ks][n]
  uint32_t* tickets;  // [row_blocks][groups + 1]
  uint32_t gsize;     // splits per fold group
  uint32_t groups;    // fold groups (1 = one flat fold)
  S* gpartials;       // [groups][n] when groups > 1
};

template <class T>
constexpr int gemv_vec_elems() {
  return mr_vec_elems<T>();
}

template <class T, class S, class F2, class Op, bool UsesX>
__global__ void __launch_bounds__(kMatThreads) gemv_kernel(const GemvArgs<T, S, F2, Op> a) {
  constexpr int VE = gemv_vec_elems<T>();
  constexpr int U = 4;
  __shared__ bool s_last;
  const uint32_t rb = blockIdx.x % a.row_blocks;
  const uint32_t s = blockIdx.x / a.row_blocks;
  const uint64_t c0 = uint64_t(s) * a.cols_per_split;
  const uint64_t c1 = c0 + a.cols_per_split < a.p ? c0 + a.cols_per_split : a.p;
  const uint64_t i0 = (uint64_t(rb) * kMatThreads + threadIdx.x) * VE;  // first row of this thread
  const T xz{};
  auto fa = [&](const T& av, const T& xv) { return a.f(av, UsesX ? xv : xz); };

  S acc[VE];
  const bool full = i0 + VE <= a.n;
  if (i0 < a.n && c0 < c1) {
    if (full && a.vec) {
      uint64_t j = c0;
      {
        T av[VE];
        load_items<T, VE>(a.A + j * a.lda + i0, av);
        const T xj = UsesX ? a.x[j] : xz;
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[e] = fa(av[e], xj);
        ++j;
      }
      for (; j + U <= c1; j += U) {
        T av[U][VE];
        T xj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          load_items<T, VE>(a.A + (j + u) * a.lda + i0, av[u]);
          xj[u] = UsesX ? a.x[j + u] : xz;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < VE; ++e) acc[e] = a.op(acc[e], fa(av[u][e], xj[u]));
      }
      for (; j < c1; ++j) {
        T av[VE];
        load_items<T, VE>(a.A + j * a.lda + i0, av);
        const T xj = UsesX ? a.x[j] : xz;
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[e] = a.op(acc[e], fa(av[e], xj));
      }
    } else {
#pragma unroll
      for (int e = 0; e < VE; ++e) {
        const uint64_t i = i0 + e;
        if (i < a.n) {
          S v = fa(a.A[c0 * a.lda + i], UsesX ? a.x[c0] : xz);
          for (uint64_t j = c0 + 1; j < c1; ++j) v = a.op(v, fa(a.A[j * a.lda + i], UsesX ? a.x[j] : xz));
          acc[e] = v;
        }
      }
    }
  }

  if (a.ks == 1) {
    if (i0 < a.n) {
      if (full && a.vec) {
        store_items<S, VE>(a.z + i0, acc);
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e)
          if (i0 + e < a.n) a.z[i0 + e] = acc[e];
      }
    }
    return;
  }
  // Partials [s][row], folded in split order in two levels so the fold tail
  // is ~2*sqrt(ks) partial rows instead of ks: the last split of each group of
  // `gsize` splits folds the group into a group partial, the last group folds
  // the group partials.  (One CTA's memory parallelism bounds a fold — 4
  // partial rows in flight per thread — and the flat fold of 56 splits was the
  // kernel's tail.)
  if (i0 < a.n) {
#pragma unroll
    for (int e = 0; e < VE; ++e)
      if (i0 + e < a.n) a.partials[uint64_t(s) * a.n + i0 + e] = acc[e];
  }
  const uint32_t grp = s / a.gsize;
  const uint32_t q0 = grp * a.gsize, q1 = q0 + a.gsize < a.ks ? q0 + a.gsize : a.ks;
  uint32_t* tk = a.tickets + uint64_t(rb) * (a.groups + 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atom_add_acq_rel_gpu(tk + grp, 1u);
    s_last = (t == q1 - q0 - 1);
    if (s_last) st_relaxed_gpu(tk + grp, 0u);
  }
  __syncthreads();
  if (!s_last) return;

  // Ordered fold of `count` partial rows (stride n) for this thread's rows.
  auto fold_rows = [&](const S* base, uint32_t count, S* out) {
    if (i0 + VE <= a.n && (sizeof(S) * VE) % 16 == 0 && is_aligned(base + i0, 16) &&
        (uint64_t(a.n) * sizeof(S)) % 16 == 0) {
      constexpr int W = int(sizeof(S) * VE) / 16;  // 16-byte words per row group
      auto load_group = [&](uint32_t q, S (&dst)[VE]) {
        uint4 w[W];
        const uint4* p = reinterpret_cast<const uint4*>(base + uint64_t(q) * a.n + i0);
#pragma unroll
        for (int k = 0; k < W; ++k)
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(w[k].x), "=r"(w[k].y), "=r"(w[k].z), "=r"(w[k].w)
                       : "l"(p + k)
                       : "memory");
        memcpy(dst, w, sizeof(S) * VE);
      };
      S acc2[VE];
      load_group(0, acc2);
      uint32_t q = 1;
      for (; q + 4 <= count; q += 4) {
        S g[4][VE];
#pragma unroll
        for (int u = 0; u < 4; ++u) load_group(q + u, g[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int e = 0; e < VE; ++e) acc2[e] = a.op(acc2[e], g[u][e]);
      }
      for (; q < count; ++q) {
        S g[VE];
        load_group(q, g);
#pragma unroll
        for (int e = 0; e < VE; ++e) acc2[e] = a.op(acc2[e], g[e]);
      }
      if (is_aligned(out + i0, 32) && (sizeof(S) * VE) % 32 == 0) {
        store_items<S, VE>(out + i0, acc2);
      } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) out[i0 + e] = acc2[e];
      }
      return;
    }
#pragma unroll
    for (int e = 0; e < VE; ++e) {
      const uint64_t i = i0 + e;
      if (i < a.n) {
        S v = ld_strong(base + i);
        for (uint32_t q = 1; q < count; ++q) v = a.op(v, ld_strong(base + uint64_t(q) * a.n + i));
        out[i] = v;
      }
    }
  };

  if (a.groups == 1) {
    fold_rows(a.partials, a.ks, a.z);
    return;
  }
  fold_rows(a.partials + uint64_t(q0) * a.n, q1 - q0, a.gpartials + uint64_t(grp) * a.n);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atom_add_acq_rel_gpu(tk + a.groups, 1u);
    s_last = (t == a.groups - 1);
    if (s_last) st_relaxed_gpu(tk + a.groups, 0u);
  }
  __syncthreads();
  if (!s_last) return;
  fold_rows(a.gpartials, a.groups, a.z);
}

// ---------------------------------------------------------------------------
// Planning + workspace (the B200 counterpart of plan_mat, primitives.hpp:220-244).

struct GevmPlan {
  uint32_t ks;
  uint64_t rows_per_split;
  uint64_t grid;
};

template <class T>
inline GevmPlan plan_gevm(uint64_t n, uint64_t p) {
  constexpr int VE = mr_vec_elems<T>();
  const uint64_t target_warps = uint64_t(device_props().sm_count) * 48;
  const uint64_t gran = uint64_t(kWarp) * VE * 4;  // rows per warp step
  uint64_t ks = p >= target_warps ? 1 : ceil_div(target_warps, p);
  const uint64_t max_ks = ceil_div(n, gran * 4);  // keep >= 4 steps per split
  if (ks > max_ks) ks = max_ks;
  if (ks < 1) ks = 1;
  if (ks > 4096) ks = 4096;
  uint64_t rps = round_up(ceil_div(n, ks), uint64_t(kWarp) * VE);
  ks = ceil_div(n, rps);
  if (ks < 1) ks = 1;
  GevmPlan pl{uint32_t(ks), rps, ceil_div(p * ks, kMatWarps)};
  return pl;
}

struct GemvPlan {
  uint32_t ks;
  uint64_t cols_per_split;
  uint32_t row_blocks;
  uint64_t grid;
  uint32_t gsize, groups;  // two-level split fold (gemv_kernel)
};

template <class T>
inline GemvPlan plan_gemv(uint64_t n, uint64_t p) {
  constexpr int VE = gemv_vec_elems<T>();
  const uint64_t row_blocks = ceil_div(n, uint64_t(kMatThreads) * VE);
  static const uint64_t per_sm = [] {
    const uint64_t v = dev_knob("FORGE_GEMV_BLOCKS_PER_SM", 3);  // measured best of 1..8 at 16384^2
    return v < 1 ? 1 : (v > 8 ? 8 : v);  // <= 8: primitives.hpp's workspace bound
  }();
  const uint64_t target_blocks = uint64_t(device_props().sm_count) * per_sm;
  uint64_t ks = row_blocks >= target_blocks ? 1 : ceil_div(target_blocks, row_blocks);
  const uint64_t max_ks = ceil_div(p, 16);  // >= 16 columns per split
  if (ks > max_ks) ks = max_ks;
  if (ks < 1) ks = 1;
  uint64_t cps = ceil_div(p, ks);
  ks = ceil_div(p, cps);
  if (ks < 1) ks = 1;
  uint32_t gsize = uint32_t(ks);
  if (ks > 8) {
    gsize = 1;
    while (uint64_t(gsize) * gsize < ks) ++gsize;  // ceil(sqrt(ks))
  }
  const uint32_t groups = uint32_t(ceil_div(ks, gsize));
  return GemvPlan{uint32_t(ks), cps, uint32_t(row_blocks), row_blocks * ks, gsize, groups};
}

// gevm_cols_kernel shape, measured at 16384² f32 (GB/s): 4 columns per warp
// 6,702 at 79 registers (3 CTAs/SM), 6,877 at <= 64 registers (4 CTAs/SM, no
// spills), 2 columns per warp 6,533; one column per warp (gevm_kernel) 6,300.
constexpr int kGevmCols = 4;
constexpr int kGevmColsMinBlocks = 4;

inline bool gevm_cols_enabled() {
  static const bool v = dev_knob("FORGE_GEVM_COLS", 1) != 0;
  return v;
}

// Plan of gevm_cols_kernel: enough (column group, row split) warps for ~14
// CTAs per SM so the last wave is nearly full.
template <class T>
inline GevmPlan plan_gevm_cols(uint64_t n, uint64_t p) {
  constexpr int VE = mr_vec_elems<T>();
  const uint64_t groups = ceil_div(p, kGevmCols);
  const uint64_t target = uint64_t(device_props().sm_count) * kMatWarps * 14;
  uint64_t ks = groups >= target ? 1 : ceil_div(target, groups);
  const uint64_t gran = uint64_t(kWarp) * VE;
  const uint64_t max_ks = ceil_div(n, gran * 8);  // >= 8 steps per split
  if (ks > max_ks) ks = max_ks;
  if (ks < 1) ks = 1;
  if (ks > 4096) ks = 4096;
  uint64_t rps = round_up(ceil_div(n, ks), gran);
  ks = ceil_div(n, rps);
  if (ks < 1) ks = 1;
  return GevmPlan{uint32_t(ks), rps, ceil_div(groups * ks, kMatWarps)};
}

template <class T, class S>
inline uint64_t gevm_ws_bytes(uint64_t n, uint64_t p) {
  const GevmPlan pl = plan_gevm<T>(n, p), pc = plan_gevm_cols<T>(n, p);
  const uint64_t ks = pl.ks > pc.ks ? pl.ks : pc.ks;
  if (ks == 1) return 256;
  return 256 + round_up(p * sizeof(uint32_t), 256) + p * ks * sizeof(S);
}

// Workspace: [256 | tickets row_blocks x (groups + 1) | partials ks x n | group partials groups x n]
template <class T, class S>
inline uint64_t gemv_ws_bytes(uint64_t n, uint64_t p) {
  GemvPlan pl = plan_gemv<T>(n, p);
  if (pl.ks == 1) return 256;
  return 256 + round_up(uint64_t(pl.row_blocks) * (pl.groups + 1) * sizeof(uint32_t), 256) +
         round_up(uint64_t(pl.ks) * n * sizeof(S), 256) + (pl.groups > 1 ? uint64_t(pl.groups) * n * sizeof(S) : 0);
}

// `lda` (>= n, 0 = n): elements between consecutive columns of A, so a block of
// a larger column-major matrix (rows [lo, lo+n) of p of its columns: A + lo +
// j0 * lda) is consumed in place — the row-block shard of vecmat and the
// sub-matrix of a sharded matvec.
template <class T, class S, class F2, class Op, bool UsesX, bool Ordered>
cudaError_t launch_gevm(const T* A, uint64_t n, uint64_t p, const T* x, S* y, const F2& f,
                        const Op& op, void* ws, cudaStream_t stream, uint64_t lda = 0) {
  if (p == 0 || n == 0) return cudaSuccess;
  if (lda == 0) lda = n;
  if (lda < n) return cudaErrorInvalidValue;
  constexpr int VE = mr_vec_elems<T>();
  const bool vec = VE > 1 && is_aligned(A, 32) && (lda * sizeof(T)) % 32 == 0 && (!UsesX || is_aligned(x, 32));
  const bool cols = !Ordered && vec && gevm_cols_enabled();
  GevmPlan pl = cols ? plan_gevm_cols<T>(n, p) : plan_gevm<T>(n, p);
  GevmArgs<T, S, F2, Op> a{A, x, y, n, p, lda, f, op, pl.ks, pl.rows_per_split, vec, nullptr, nullptr};
  if (pl.ks > 1) {
    char* w = static_cast<char*>(ws) + 256;
    a.tickets = reinterpret_cast<uint32_t*>(w);
    const uint64_t tbytes = round_up(p * sizeof(uint32_t), 256);
    a.partials = reinterpret_cast<S*>(w + tbytes);
    if (const cudaError_t e = ws_claim(ws, ws_tag(3, tbytes), 256 + tbytes, stream,
                                       256 + tbytes + uint64_t(pl.ks) * p * sizeof(S));
        e != cudaSuccess)
      return e;
  }
  if constexpr (!Ordered) {
    if (cols) {
      gevm_cols_kernel<T, S, F2, Op, UsesX, kGevmCols, kGevmColsMinBlocks>
          <<<uint32_t(pl.grid), kMatThreads, 0, stream>>>(a);
      return cudaGetLastError();
    }
  }
  gevm_kernel<T, S, F2, Op, UsesX, Ordered><<<uint32_t(pl.grid), kMatThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

template <class T, class S, class F2, class Op, bool UsesX>
cudaError_t launch_gemv(const T* A, uint64_t n, uint64_t p, const T* x, S* z, const F2& f,
                        const Op& op, void* ws, cudaStream_t stream, uint64_t lda = 0) {
  if (p == 0 || n == 0) return cudaSuccess;
  if (lda == 0) lda = n;
  if (lda < n) return cudaErrorInvalidValue;
  constexpr int VE = gemv_vec_elems<T>();
  GemvPlan pl = plan_gemv<T>(n, p);
  GemvArgs<T, S, F2, Op> a{A,  x,     z,     n,     p,       lda,     f, op, pl.ks, pl.cols_per_split, pl.row_blocks,
                           false, nullptr, nullptr, pl.gsize, pl.groups, nullptr};
  a.vec = VE > 1 && is_aligned(A, 32) && (lda * sizeof(T)) % 32 == 0 && is_aligned(z, 32);
  if (pl.ks > 1) {
    char* w = static_cast<char*>(ws) + 256;
    a.tickets = reinterpret_cast<uint32_t*>(w);
    const uint64_t tbytes = round_up(uint64_t(pl.row_blocks) * (pl.groups + 1) * sizeof(uint32_t), 256);
    const uint64_t extent = 256 + tbytes + round_up(uint64_t(pl.ks) * n * sizeof(S), 256) +
                            (pl.groups > 1 ? uint64_t(pl.groups) * n * sizeof(S) : 0);
    if (const cudaError_t e = ws_claim(ws, ws_tag(4, pl.row_blocks, pl.groups), 256 + tbytes, stream, extent);
        e != cudaSuccess)
      return e;
    w += tbytes;
    a.partials = reinterpret_cast<S*>(w);
    w += round_up(uint64_t(pl.ks) * n * sizeof(S), 256);
    if (pl.groups > 1) a.gpartials = reinterpret_cast<S*>(w);
  }
  gemv_kernel<T, S, F2, Op, UsesX><<<uint32_t(pl.grid), kMatThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace forge::cuda
