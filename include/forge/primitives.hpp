// forge/primitives.hpp — the drop-in primitive API, executed by sm_100a kernels.
//
// Same names, signatures, argument meaning and error behaviour as
// /root/reference/proj/include/forge/primitives.hpp:
//   ArchParams (:16-60)  MutationFlags / RunOptions (:64-84)
//   SemiringSpec / make_semiring (:92-104)  validate_reduce_op (:108-118)
//   OptVal helpers (:124-146)  Primitive / TileFlag / Workspace (:176-195)
//   scan_tiles (:197-200)  required_workspace / make_*_workspace (:246-300)
//   vcopy (:305-341)  mapreduce (:348-431)  scan (:440-603)
//   matvec (:776-791)  vecmat (:795-807)  mapreduce_2d (:809-836)
// The bodies launch the kernels of forge/cuda/*.cuh on the Machine's stream
// and return a LaunchReport whose wall_seconds is the CUDA-event time of the
// device work.  User functors must be device-callable (__host__ __device__
// functor structs, or __device__ lambdas with --extended-lambda) because they
// are inlined into the kernels; a translation unit using these templates must
// therefore be compiled by nvcc.  Plain C / C++ / FFI users reach the fixed
// operator menu through include/forge.h instead.
//
// B200 deviations (all documented in DESIGN.md):
//   * warp_width 64 raises ErrorCode::Unsupported (declared by the reference,
//     error.hpp:18, never raised there).
//   * The geometry fields of ArchParams are validated like the reference but
//     the kernels choose their own tiles / grids; RunOptions::backend,
//     tuning are accepted and ignored (there is no simulator and no CPU
//     fallback); a non-zero schedule.seed perturbs the scan's schedule the B200
//     way (1/8 of the tiles, chosen by the seed, publish 20 us late:
//     cuda::ScanTestHooks) — results are unchanged, only slower.  mutate.relax_scan_flag selects the scan ablation (tile
//     states of earlier launches accepted: a broken publication protocol the
//     stress tests must catch); relax_mapreduce_flag is accepted and ignored
//     (the mapreduce never waits on another block's flag).
//   * Workspaces use the B200 layouts (forge/cuda/*.cuh): they are zeroed once
//     at creation and self-reset, so no fill_zero happens per launch; a
//     workspace moved to another layout (another primitive, another matrix
//     plan) is re-zeroed by the library first (cuda::ws_claim).
#pragma once

#include <algorithm>
#include <cstddef>
#include <optional>
#include <span>
#include <vector>

#include "forge/intrinsics.hpp"
#include "forge/machine.hpp"

#ifdef __CUDACC__
#include "forge/cuda/copy.cuh"
#include "forge/cuda/matrix.cuh"
#include "forge/cuda/reduce.cuh"
#include "forge/cuda/scan.cuh"
#endif

#ifdef __CUDACC__
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (ranges around primitive calls)
#endif

namespace forge::prim {

using intr::View;

struct ArchParams {
  uint32_t warp_width = 32;
  uint32_t mapreduce_blocks = 100;
  uint32_t threads_per_block = 256;
  uint32_t nitem_scan = 16;
  uint32_t nitem_copy = 4;
  uint32_t lookback_window = 0;  // 0 = warp_width
  uint32_t matvec_wide_warp_cols = 4;
  uint32_t matvec_wide_block_threads = 128;
  uint64_t matvec_wide_min_outputs = 0;  // 0 = 4*blocks*(tpb/warp)*cols

  ArchParams normalized() const {
    ArchParams p = *this;
    if (p.lookback_window == 0) p.lookback_window = p.warp_width;
    if (p.matvec_wide_min_outputs == 0 && p.warp_width != 0)
      p.matvec_wide_min_outputs = 4ull * p.mapreduce_blocks * (p.threads_per_block / p.warp_width) *
                                  p.matvec_wide_warp_cols;
    p.validate();
    return p;
  }

  void validate() const {
    const auto nitem_ok = [](uint32_t v) { return v == 1 || v == 2 || v == 4 || v == 8 || v == 16; };
    if (warp_width != 32 && warp_width != 64)
      raise(ErrorCode::InvalidArgument, "warp_width must be 32 or 64");
    if (warp_width != 32)
      raise(ErrorCode::Unsupported, "warp_width 64 (AMD wavefronts) is not a B200 configuration");
    if (threads_per_block == 0 || threads_per_block % warp_width != 0 ||
        threads_per_block > warp_width * warp_width)
      raise(ErrorCode::InvalidArgument,
            "threads_per_block must be a multiple of warp_width, at most warp_width^2");
    if (mapreduce_blocks == 0) raise(ErrorCode::InvalidArgument, "mapreduce_blocks");
    if (!nitem_ok(nitem_scan) || !nitem_ok(nitem_copy))
      raise(ErrorCode::InvalidNitem, "nitem must be one of {1,2,4,8,16}");
    if (lookback_window != 0 && lookback_window != warp_width)
      raise(ErrorCode::InvalidArgument, "lookback_window must equal warp_width");
    if (matvec_wide_block_threads == 0 || matvec_wide_block_threads % warp_width != 0)
      raise(ErrorCode::InvalidArgument, "matvec_wide_block_threads");
    if (matvec_wide_warp_cols == 0 || matvec_wide_warp_cols > 8)
      raise(ErrorCode::InvalidArgument, "matvec_wide_warp_cols must be in 1..8");
  }
};

struct MutationFlags {
  bool relax_scan_flag = false;
  bool relax_mapreduce_flag = false;
};

struct RunOptions {
  Backend backend = Backend::Simulator;  // accepted, ignored: the GPU executes
  ScheduleSeed schedule{};
  SimTuning tuning{};
  TraceSink* trace = nullptr;  // one record per kernel launch
  MutationFlags mutate{};
};

inline LaunchOptions to_launch_options(const RunOptions& o) {
  LaunchOptions lo;
  lo.backend = o.backend;
  lo.schedule = o.schedule;
  lo.tuning = o.tuning;
  lo.trace = o.trace;
  return lo;
}

template <class F, class S, class Op>
struct SemiringSpec {
  F map;
  Op op;
  std::optional<S> identity;
  bool commutative = false;
};

template <class S, class F, class Op>
SemiringSpec<F, S, Op> make_semiring(F map, Op op, std::optional<S> identity, bool commutative) {
  return SemiringSpec<F, S, Op>{map, op, identity, commutative};
}

template <class S, class Op, class Gen, class Eq>
bool validate_reduce_op(const Op& op, const std::optional<S>& identity, bool commutative, Gen&& gen,
                        Eq&& eq, int samples = 256) {
  for (int i = 0; i < samples; ++i) {
    const S a = gen(), b = gen(), c = gen();
    if (!eq(op(op(a, b), c), op(a, op(b, c)))) return false;
    if (commutative && !eq(op(a, b), op(b, a))) return false;
    if (identity && (!eq(op(*identity, a), a) || !eq(op(a, *identity), a))) return false;
  }
  return true;
}

template <class S>
struct OptVal {
  S value;
  uint8_t valid;
};
template <class S>
inline OptVal<S> opt_none() {
  return OptVal<S>{S{}, 0};
}
template <class S>
inline OptVal<S> opt_of(const S& v) {
  return OptVal<S>{v, 1};
}
template <class Op, class S>
inline OptVal<S> opt_combine(const Op& op, const OptVal<S>& a, const OptVal<S>& b) {
  if (!a.valid) return b;
  if (!b.valid) return a;
  return OptVal<S>{op(a.value, b.value), 1};
}

enum class Primitive : uint8_t { Scan, MapReduce, MatVec, VecMat, VCopy, MapReduce2d };
enum class TileFlag : uint8_t { Invalid = 0, Partial = 1, Prefix = 2 };
enum class ReduceAxis : uint8_t { Rows, Cols };

// Workspace handles (primitives.hpp:180-195).  B200 use of the fields:
//   tile_flag : scan control words + per-tile {status, carry} state words
//   partials  : mapreduce / matrix partials and arrival tickets (bytes)
//   result    : mapreduce device result
//   tiles     : scan tile capacity; slots: byte capacity of `partials`
struct Workspace {
  BufferId tile_aggregate = -1;
  BufferId tile_prefix = -1;
  BufferId tile_flag = -1;
  BufferId partials = -1;
  BufferId flags = -1;
  BufferId result = -1;
  uint64_t tiles = 0;
  uint64_t slots = 0;

  void release(Machine& m) {
    for (BufferId id : {tile_aggregate, tile_prefix, tile_flag, partials, flags, result})
      if (id >= 0) m.destroy_buffer(id);
    *this = Workspace{};
  }
};

// Reference tile arithmetic, kept for the API.
inline uint64_t scan_tiles(uint64_t n, const ArchParams& p) {
  const uint64_t tile = uint64_t(p.threads_per_block) * p.nitem_scan;
  return (n + tile - 1) / tile;
}

// Matrix primitive geometry (primitives.hpp:202-244), kept for the API: the
// same fields and the reference's own formulas, so code that sizes or logs a
// plan keeps compiling and gets the same numbers.  The sm_100a kernels plan
// their own launches; b200_plan_mat<T>() (nvcc TUs) reports that geometry in
// the same struct.
struct MatPlan {
  bool wide = false;
  uint64_t nb = 1;            // tall: slices per output (B200: row / column splits)
  uint64_t rows_per_slice = 0;
  uint64_t grid_outputs = 0;  // tall: outputs in flight
  uint64_t groups = 0;        // wide: output groups per grid pass
  LaunchConfig cfg;
  uint64_t slots = 0;         // partial slots (nb > 1)
};

inline uint64_t tall_slices(uint64_t reduce_len, const ArchParams& p) {
  const uint64_t per_slice = uint64_t(p.threads_per_block) * p.nitem_copy * 8;
  return std::clamp<uint64_t>((reduce_len + per_slice - 1) / per_slice, 1, p.mapreduce_blocks);
}

inline MatPlan plan_mat(uint64_t reduce_len, uint64_t outputs, bool commutative, const ArchParams& params) {
  const ArchParams p = params.normalized();
  MatPlan plan;
  const uint32_t V = p.nitem_copy;
  const bool order_free = commutative || reduce_len <= V;
  if (outputs >= p.matvec_wide_min_outputs && order_free) {
    plan.wide = true;
    const uint32_t warps = p.matvec_wide_block_threads / p.warp_width;
    const uint64_t per_block = uint64_t(warps) * p.matvec_wide_warp_cols;
    const uint64_t needed = (outputs + per_block - 1) / per_block;
    plan.groups = needed;
    plan.cfg.num_blocks = uint32_t(std::min<uint64_t>(needed, 2ull * p.mapreduce_blocks));
    plan.cfg.threads_per_block = p.matvec_wide_block_threads;
  } else {
    plan.nb = tall_slices(reduce_len, p);
    plan.rows_per_slice = (reduce_len + plan.nb - 1) / plan.nb;
    plan.grid_outputs = std::min<uint64_t>(outputs, std::max<uint64_t>(1, 4ull * p.mapreduce_blocks / plan.nb));
    plan.cfg.num_blocks = uint32_t(plan.nb * plan.grid_outputs);
    plan.cfg.threads_per_block = p.threads_per_block;
    if (plan.nb > 1) plan.slots = plan.nb * outputs;
  }
  plan.cfg.warp_width = p.warp_width;
  return plan;
}

namespace detail {

inline uint64_t rup(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// Scan workspace bound for an S of `s_size` bytes (cuda::ScanWs, which this
// mirrors with the carry bounded by 2 * sizeof(S): f32 sums carry in f64):
// the smem kernel's tiles of a sizeof(S)-byte T at full 256-byte slots, or the
// general kernel's tiles (256 x 64 bytes of S) at packed slots, whichever is
// larger.  Smaller workspaces (down to packed slots) are accepted too.
inline uint64_t b200_scan_general_tile(uint32_t s_size) {
  return 256 * std::clamp<uint64_t>(64 / std::max<uint32_t>(s_size, 1), 1, 16);
}
inline uint64_t b200_scan_sized_tile(uint32_t s_size) {
  if (s_size >= 16) return 2 * 256 * 8;
  return 256 * std::max<uint64_t>(128 / std::max<uint32_t>(s_size, 1), 1);
}
inline uint64_t b200_state_min_bytes(uint32_t accum_size) {  // packed slot: every 32-bit chunk of the carry
  const uint64_t words = (2ull * accum_size + 3) / 4;
  uint64_t stride = 1;
  while (stride < words) stride <<= 1;
  return stride * 8;
}
inline uint64_t b200_state_group_tiles(uint32_t accum_size) {  // tile states per 32-byte group
  const uint64_t words = b200_state_min_bytes(accum_size) / 8;
  return words <= 4 ? 4 / words : 1;
}
inline uint64_t b200_sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 148;
  return uint64_t(sms);
}
inline uint64_t b200_scan_ws_base(uint64_t n, uint32_t accum_size) {  // single-pass kernels
  const uint64_t P = b200_state_group_tiles(accum_size);
  const uint64_t sized_tiles = std::max<uint64_t>((n + b200_scan_sized_tile(accum_size) - 1) /
                                                      b200_scan_sized_tile(accum_size), 1);
  const uint64_t full = 256 + (sized_tiles + P - 1) / P *
                                  std::max<uint64_t>(b200_state_min_bytes(accum_size) * P, 256);
  const uint64_t packed = 256 + 32 +  // + one partial 32-byte group
                          std::max<uint64_t>((n + b200_scan_general_tile(accum_size) - 1) /
                                                 b200_scan_general_tile(accum_size), 1) *
                              b200_state_min_bytes(accum_size);
  return std::max(full, packed);
}
inline uint64_t b200_scan_ws_bytes(uint64_t n, uint32_t accum_size) {
  uint64_t lag = 0;  // the lagged kernel's layout (cuda::LagWs) for a sizeof(S)-byte T
  if (accum_size <= 16 && (accum_size & (accum_size - 1)) == 0) {
    const uint64_t tile = 256 * (128 / accum_size);
    const uint64_t tiles = n / tile;
    if (tiles >= std::max<uint64_t>(3 * (b200_sm_count() * 4), 128)) {  // cuda::lag_min_tiles()
      const uint64_t smb = b200_state_min_bytes(accum_size);
      lag = 256 + rup(tiles * smb, 256) + rup((tiles + 31) / 32 * smb, 256) + 256 +
            b200_scan_ws_base(tile, accum_size);
    }
  }
  return std::max(b200_scan_ws_base(n, accum_size), lag);
}
inline uint64_t b200_mapreduce_ws_bytes(uint32_t accum_size) {
  const uint64_t grid = b200_sm_count() * 4;
  return 256 + rup(grid * std::max<uint32_t>(2 * accum_size, 8), 256) + rup(grid * 4, 256);
}
// Matrix partials: generous bound covering both kernels' plans for (reduce_len, outputs).
inline uint64_t b200_mat_ws_bytes(uint32_t accum_size, uint64_t reduce_len, uint64_t outputs) {
  const uint64_t sms = b200_sm_count();
  // gevm: one-column plan ks <= ceil(sms*48 / outputs); column-group plan (4
  // columns per warp, ~14 CTAs of 8 warps per SM) ks <= ceil(sms*448 / outputs);
  // p tickets, outputs*ks partials
  const uint64_t outs1 = std::max<uint64_t>(outputs, 1);
  const uint64_t ks_v = std::max<uint64_t>(1, std::max((sms * 48 + outs1 - 1) / outs1, (sms * 448 + outs1 - 1) / outs1));
  const uint64_t gevm = 256 + rup(outputs * 4, 256) + outputs * ks_v * accum_size;
  // gemv: ks <= sms*8 splits (3/SM default, FORGE_GEMV_BLOCKS_PER_SM <= 8), row
  // blocks of >= 256 rows, each with (groups + 1) tickets, groups <= ceil(sqrt(ks)),
  // ks*outputs split partials + groups*outputs group partials
  const uint64_t ks_m = std::min<uint64_t>(sms * 8, std::max<uint64_t>(1, (reduce_len + 15) / 16));
  uint64_t groups = 1;
  while (groups * groups < ks_m) ++groups;
  const uint64_t row_blocks = (outputs + 255) / 256;
  const uint64_t gemv = 256 + rup(row_blocks * (groups + 1) * 4, 256) + rup(ks_m * outputs * accum_size, 256) +
                        groups * outputs * accum_size;
  return rup(std::max(gevm, gemv), 256);
}

}  // namespace detail

inline uint64_t required_workspace(Primitive prim, uint32_t accum_size, uint64_t n, uint64_t p_cols,
                                   const ArchParams& params_in) {
  (void)params_in.normalized();
  switch (prim) {
    case Primitive::Scan:
      return detail::b200_scan_ws_bytes(n, accum_size);
    case Primitive::MapReduce:
      return detail::b200_mapreduce_ws_bytes(accum_size) + 256;
    case Primitive::MatVec:
    case Primitive::MapReduce2d:
      return detail::b200_mat_ws_bytes(accum_size, n, p_cols);
    case Primitive::VecMat:
      return detail::b200_mat_ws_bytes(accum_size, p_cols, n);
    case Primitive::VCopy:
      return 0;
  }
  return 0;
}

template <class S>
Workspace make_scan_workspace(Machine& m, uint64_t n, const ArchParams& params) {
  (void)params.normalized();
  Workspace ws;
  const uint64_t bytes = detail::b200_scan_ws_bytes(n, sizeof(S));
  ws.tiles = (n + detail::b200_scan_general_tile(sizeof(S)) - 1) / detail::b200_scan_general_tile(sizeof(S));
  ws.tile_flag = intr::create_buffer<uint8_t>(m, bytes, 256);
  return ws;
}

template <class S>
Workspace make_mapreduce_workspace(Machine& m, const ArchParams& params) {
  (void)params.normalized();
  Workspace ws;
  ws.slots = detail::b200_mapreduce_ws_bytes(sizeof(S));
  ws.partials = intr::create_buffer<uint8_t>(m, ws.slots, 256);
  ws.result = intr::create_buffer<uint8_t>(m, detail::rup(sizeof(S), 16) + 16, 256);
  return ws;
}

template <class S>
Workspace make_mat_workspace(Machine& m, uint64_t reduce_len, uint64_t outputs,
                             const ArchParams& params) {
  (void)params.normalized();
  Workspace ws;
  ws.slots = std::max(detail::b200_mat_ws_bytes(sizeof(S), reduce_len, outputs),
                      detail::b200_mat_ws_bytes(sizeof(S), outputs, reduce_len));
  ws.partials = intr::create_buffer<uint8_t>(m, ws.slots, 256);
  return ws;
}

#ifdef __CUDACC__

// The geometry the sm_100a kernels actually launch for matvec (gevm, fold down
// the n rows of each of p columns) or vecmat (gemv, fold across the p columns
// of each of n rows), in the reference's MatPlan terms: `wide` = the
// column-group / row-per-thread kernels (commutative ops on aligned data), `nb`
// = splits of the fold per output, `slots` = partials in the workspace.
template <class T>
MatPlan b200_plan_mat(Primitive prim, uint64_t n, uint64_t p_cols, bool commutative) {
  MatPlan plan;
  plan.cfg.warp_width = 32;
  plan.cfg.threads_per_block = cuda::kMatThreads;
  if (prim == Primitive::VecMat) {
    const cuda::GemvPlan g = cuda::plan_gemv<T>(n, p_cols);
    plan.wide = true;
    plan.nb = g.ks;
    plan.rows_per_slice = g.cols_per_split;
    plan.groups = g.row_blocks;
    plan.grid_outputs = n;
    plan.cfg.num_blocks = uint32_t(g.grid);
    plan.slots = g.ks > 1 ? g.ks * n : 0;
    return plan;
  }
  const bool cols = commutative && cuda::gevm_cols_enabled();
  const cuda::GevmPlan g = cols ? cuda::plan_gevm_cols<T>(n, p_cols) : cuda::plan_gevm<T>(n, p_cols);
  plan.wide = cols;
  plan.nb = g.ks;
  plan.rows_per_slice = g.rows_per_split;
  plan.groups = cols ? cuda::ceil_div(p_cols, cuda::kGevmCols) : p_cols;
  plan.grid_outputs = p_cols;
  plan.cfg.num_blocks = uint32_t(g.grid);
  plan.slots = g.ks > 1 ? g.ks * p_cols : 0;
  return plan;
}

namespace detail {

// NVTX range around every primitive call (header-only NVTX v3: a no-op unless
// a profiler such as nsys injects itself).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class Fn>
LaunchReport run_timed(Machine& m, const RunOptions& opt, const char* name, uint64_t elems,
                       Fn&& launch) {
  NvtxRange range(name);
  LaunchReport rep;
  rep.buffers.resize(m.buffer_count());
  uint64_t launches = 0;
  m.begin_timing();
  cudaError_t e = launch(launches);
  double secs = 0.0;
  const cudaError_t e2 = m.end_timing(secs);
  if (e == cudaSuccess) e = e2;
  rep.steps = launches;
  rep.wall_seconds = secs;
  if (e != cudaSuccess) {
    rep.ok = false;
    rep.fault.kind = FaultKind::Internal;
    rep.fault.detail = std::string(name) + ": " + cudaGetErrorString(e);
    return rep;
  }
  rep.ok = true;
  if (opt.trace)
    opt.trace->on_event(TraceEvent{0, 0, 0, name, -1, elems, MemoryOrdering::Relaxed, 0});
  return rep;
}

inline void count_load(LaunchReport& r, BufferId b, uint64_t n) {
  if (b >= 0 && size_t(b) < r.buffers.size()) {
    r.buffers[b].load_events += n;
    r.buffers[b].load_elems += n;
  }
}
inline void count_store(LaunchReport& r, BufferId b, uint64_t n) {
  if (b >= 0 && size_t(b) < r.buffers.size()) {
    r.buffers[b].store_events += n;
    r.buffers[b].store_elems += n;
  }
}

inline uint64_t buffer_bytes(const Machine& m, BufferId id) {
  return id < 0 ? 0 : m.buffer_length(id) * m.buffer_elem_size(id);
}

// f(x, a) -> f(a) and f(a, x) -> f(a): the unary map lifted for mapreduce_2d
// (primitives.hpp:819-832).
template <class F>
struct LiftSecond {
  F f;
  template <class T>
  __host__ __device__ __forceinline__ auto operator()(const T&, const T& a) const { return f(a); }
};
template <class F>
struct LiftFirst {
  F f;
  template <class T>
  __host__ __device__ __forceinline__ auto operator()(const T& a, const T&) const { return f(a); }
};

}  // namespace detail

template <class T>
LaunchReport vcopy(Machine& m, View<T> src, View<T> dst, uint32_t nitem, const ArchParams& params,
                   const RunOptions& opt = {}) {
  (void)params.normalized();
  if (nitem != 1 && nitem != 2 && nitem != 4 && nitem != 8 && nitem != 16)
    raise(ErrorCode::InvalidNitem, "vcopy nitem");
  if (src.length != dst.length) raise(ErrorCode::DimensionMismatch, "vcopy lengths differ");
  const uint64_t n = src.length;
  if (n == 0) {
    LaunchReport rep;
    rep.ok = true;
    rep.buffers.resize(m.buffer_count());
    return rep;
  }
  const T* sp = intr::view_ptr(m, src);
  T* dp = intr::view_ptr(m, dst);
  LaunchReport rep = detail::run_timed(m, opt, "vcopy", n, [&](uint64_t& k) {
    k = 1;
    return cuda::launch_strided_copy<T>(sp, src.stride, dp, dst.stride, n, m.stream());
  });
  detail::count_load(rep, src.buf, n);
  detail::count_store(rep, dst.buf, n);
  return rep;
}

template <class T, class S, class F, class Op>
LaunchReport mapreduce(Machine& m, const SemiringSpec<F, S, Op>& spec, View<T> src, Workspace& ws,
                       const ArchParams& params, S* out, const RunOptions& opt = {}) {
  (void)params.normalized();
  if (!spec.commutative)
    raise(ErrorCode::InvalidArgument, "mapreduce requires an operator declared commutative");
  const uint64_t n = src.length;
  if (n == 0) {
    if (!spec.identity) raise(ErrorCode::MissingIdentity, "empty mapreduce needs an identity");
    *out = *spec.identity;
    LaunchReport rep;
    rep.ok = true;
    rep.buffers.resize(m.buffer_count());
    return rep;
  }
  if (ws.partials < 0 || ws.result < 0 ||
      detail::buffer_bytes(m, ws.partials) < detail::b200_mapreduce_ws_bytes(sizeof(S)) ||
      detail::buffer_bytes(m, ws.result) < detail::rup(sizeof(S), 16) + sizeof(uint32_t))
    raise(ErrorCode::WorkspaceTooSmall, "mapreduce workspace");
  const T* sp = intr::view_ptr(m, src);
  char* wsp = static_cast<char*>(m.device_ptr(ws.partials));
  S* res = static_cast<S*>(m.device_ptr(ws.result));
  uint32_t* has = reinterpret_cast<uint32_t*>(static_cast<char*>(m.device_ptr(ws.result)) +
                                              detail::rup(sizeof(S), 16));
  LaunchReport rep = detail::run_timed(m, opt, "mapreduce", n, [&](uint64_t& k) {
    k = 1;
    return cuda::launch_mapreduce<T, S, F, Op>(sp, n, src.stride, spec.map, spec.op, res, has, wsp,
                                               m.stream());
  });
  detail::count_load(rep, src.buf, n);
  if (rep.ok) {
    std::vector<std::byte> tmp(sizeof(S));
    m.read_bytes(ws.result, 0, tmp);
    std::memcpy(out, tmp.data(), sizeof(S));
  }
  return rep;
}

template <class T, class S, class F, class Op>
LaunchReport scan(Machine& m, const SemiringSpec<F, S, Op>& spec, View<T> src, View<S> dst,
                  bool inclusive, Workspace& ws, const ArchParams& params,
                  const RunOptions& opt = {}) {
  (void)params.normalized();
  if (src.length != dst.length) raise(ErrorCode::DimensionMismatch, "scan lengths differ");
  if (!inclusive && !spec.identity)
    raise(ErrorCode::MissingIdentity, "exclusive scan needs an identity");
  const uint64_t n = src.length;
  if (n == 0) {
    LaunchReport rep;
    rep.ok = true;
    rep.buffers.resize(m.buffer_count());
    return rep;
  }
  using WsT = cuda::ScanWs<T, S, Op>;
  const uint64_t ws_bytes = detail::buffer_bytes(m, ws.tile_flag);
  if (ws.tile_flag < 0 || ws_bytes < WsT::min_bytes_for(cuda::ceil_div(n, WsT::kTileGeneral)))
    raise(ErrorCode::WorkspaceTooSmall, "scan workspace");
  const T* sp = intr::view_ptr(m, src);
  S* dp = intr::view_ptr(m, dst);
  void* wsp = m.device_ptr(ws.tile_flag);
  const S ident = spec.identity.value_or(S{});
  LaunchReport rep = detail::run_timed(m, opt, "scan", n, [&](uint64_t& k) {
    k = 1;
    return cuda::launch_scan<T, S, F, Op>(sp, src.stride, dp, dst.stride, n, inclusive, spec.map, spec.op, ident,
                                          nullptr, nullptr, wsp, ws_bytes, m.stream(),
                                          cuda::ScanTestHooks{opt.mutate.relax_scan_flag, opt.schedule.seed,
                                                              opt.schedule.seed ? 20000u : 0u});
  });
  detail::count_load(rep, src.buf, n);
  detail::count_store(rep, dst.buf, n);
  return rep;
}

namespace detail {

// Shared body of matvec / vecmat: output fill for empty folds, strided
// x/out staging through machine scratch, launch.
template <bool IsGevm, class T, class S, class F2, class Op>
LaunchReport run_matrix(Machine& m, const SemiringSpec<F2, S, Op>& spec, View<T> A, uint64_t n,
                        uint64_t p_cols, View<T> x, View<S> out, Workspace& ws,
                        const RunOptions& opt, bool uses_vector) {
  const uint64_t outputs = IsGevm ? p_cols : n;
  const uint64_t reduce_len = IsGevm ? n : p_cols;
  LaunchReport rep;
  rep.buffers.resize(m.buffer_count());
  if (outputs == 0) {
    rep.ok = true;
    return rep;
  }
  if (reduce_len == 0) {
    if (!spec.identity) raise(ErrorCode::MissingIdentity, "empty reduction needs an identity");
    std::vector<S> fill(outputs, *spec.identity);
    if (out.contiguous()) {
      m.write(out.buf, std::span<const S>(fill), out.offset);
    } else {
      for (uint64_t i = 0; i < outputs; ++i)
        m.write(out.buf, std::span<const S>(&fill[i], 1), out.index_of(i));
    }
    rep.ok = true;
    return rep;
  }
  const uint64_t need = IsGevm ? cuda::gevm_ws_bytes<T, S>(n, p_cols) : cuda::gemv_ws_bytes<T, S>(n, p_cols);
  if (need > 256 && (ws.partials < 0 || buffer_bytes(m, ws.partials) < need))
    raise(ErrorCode::WorkspaceTooSmall, "matrix primitive workspace");
  void* wsp = ws.partials >= 0 ? m.device_ptr(ws.partials) : nullptr;
  const T* Ap = intr::view_ptr(m, A);
  const T* xp = uses_vector ? intr::view_ptr(m, x) : nullptr;
  S* op_ = intr::view_ptr(m, out);
  // Stage strided operands contiguously (the kernels read x / write out densely).
  const size_t xbytes = uses_vector && !x.contiguous() ? rup(reduce_len * sizeof(T), 256) : 0;
  const size_t obytes = !out.contiguous() ? rup(outputs * sizeof(S), 256) : 0;
  char* scratch = (xbytes + obytes) ? static_cast<char*>(m.scratch(xbytes + obytes)) : nullptr;
  T* xs = xbytes ? reinterpret_cast<T*>(scratch) : nullptr;
  S* os = obytes ? reinterpret_cast<S*>(scratch + xbytes) : nullptr;
  const bool ordered = !spec.commutative;
  rep = run_timed(m, opt, IsGevm ? "matvec" : "vecmat", n * p_cols, [&](uint64_t& k) {
    cudaError_t e = cudaSuccess;
    const T* xk = xp;
    if (xs) {
      e = cuda::launch_strided_copy<T>(xp, x.stride, xs, 1, reduce_len, m.stream());
      xk = xs;
      ++k;
    }
    S* ok = os ? os : op_;
    if (e == cudaSuccess) {
      ++k;
      if constexpr (IsGevm) {
        if (uses_vector)
          e = ordered ? cuda::launch_gevm<T, S, F2, Op, true, true>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream())
                      : cuda::launch_gevm<T, S, F2, Op, true, false>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream());
        else
          e = ordered ? cuda::launch_gevm<T, S, F2, Op, false, true>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream())
                      : cuda::launch_gevm<T, S, F2, Op, false, false>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream());
      } else {
        if (uses_vector)
          e = cuda::launch_gemv<T, S, F2, Op, true>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream());
        else
          e = cuda::launch_gemv<T, S, F2, Op, false>(Ap, n, p_cols, xk, ok, spec.map, spec.op, wsp, m.stream());
      }
    }
    if (e == cudaSuccess && os) {
      e = cuda::launch_strided_copy<S>(os, 1, op_, out.stride, outputs, m.stream());
      ++k;
    }
    return e;
  });
  count_load(rep, A.buf, n * p_cols);
  if (uses_vector) count_load(rep, x.buf, reduce_len);
  count_store(rep, out.buf, outputs);
  return rep;
}

}  // namespace detail

template <class T, class S, class F2, class Op>
LaunchReport matvec(Machine& m, const SemiringSpec<F2, S, Op>& spec, View<T> A, uint64_t n,
                    uint64_t p_cols, View<T> x, View<S> y, Workspace& ws, const ArchParams& params,
                    const RunOptions& opt = {}, bool uses_vector = true) {
  (void)params.normalized();
  if (A.length != n * p_cols || (uses_vector && x.length != n) || y.length != p_cols)
    raise(ErrorCode::DimensionMismatch, "matvec shapes");
  if (!A.contiguous()) raise(ErrorCode::InvalidArgument, "matvec needs contiguous A");
  return detail::run_matrix<true>(m, spec, A, n, p_cols, x, y, ws, opt, uses_vector);
}

template <class T, class S, class F2, class Op>
LaunchReport vecmat(Machine& m, const SemiringSpec<F2, S, Op>& spec, View<T> A, uint64_t n,
                    uint64_t p_cols, View<T> x, View<S> z, Workspace& ws, const ArchParams& params,
                    const RunOptions& opt = {}, bool uses_vector = true) {
  (void)params.normalized();
  if (A.length != n * p_cols || (uses_vector && x.length != p_cols) || z.length != n)
    raise(ErrorCode::DimensionMismatch, "vecmat shapes");
  if (!A.contiguous()) raise(ErrorCode::InvalidArgument, "vecmat needs contiguous A");
  return detail::run_matrix<false>(m, spec, A, n, p_cols, x, z, ws, opt, uses_vector);
}

template <class T, class S, class F, class Op>
LaunchReport mapreduce_2d(Machine& m, const SemiringSpec<F, S, Op>& spec, View<T> A, uint64_t n,
                          uint64_t p_cols, ReduceAxis axis, View<S> out, Workspace& ws,
                          const ArchParams& params, const RunOptions& opt = {}) {
  View<T> none{A.buf, 0, 0, 1};
  if (axis == ReduceAxis::Rows) {
    SemiringSpec<detail::LiftSecond<F>, S, Op> lifted{{spec.map}, spec.op, spec.identity, spec.commutative};
    return matvec<T, S>(m, lifted, A, n, p_cols, none, out, ws, params, opt, /*uses_vector=*/false);
  }
  SemiringSpec<detail::LiftFirst<F>, S, Op> lifted{{spec.map}, spec.op, spec.identity, spec.commutative};
  return vecmat<T, S>(m, lifted, A, n, p_cols, none, out, ws, params, opt, /*uses_vector=*/false);
}

#endif  // __CUDACC__

}  // namespace forge::prim

namespace forge::intr {

// Descriptor of OptVal<S> (primitives.hpp:840-853): the value at 0, the valid
// byte after it, the C++ size (padding included).
template <class S>
struct TypeOf<prim::OptVal<S>> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::struct_of(
        {{descriptor_of<S>(), 0},
         {TypeDescriptor::primitive(Scalar::U8), uint32_t(offsetof(prim::OptVal<S>, valid))}},
        uint32_t(sizeof(prim::OptVal<S>)));
    return d;
  }
};

}  // namespace forge::intr
