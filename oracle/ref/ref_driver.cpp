// ref_driver.cpp — extern "C" entry points over the UNMODIFIED reference
// primitives (/root/reference/proj/include/forge/primitives.hpp) running on the
// reference's own CPU VM (Simulator or Threads backend, machine.cpp:1025-1151).
//
// ORACLE / CPU-BASELINE SUPPORT ONLY.  Built by oracle/ref/build_ref.py into
// oracle/_ref/libforge_ref.so; loaded by tests/ (parity pinning of the oracle
// restatement) and by bench.py --impl reference / cpu_baseline.  Never linked
// into the product.
//
// The operator menu follows include/forge.h's forge_op.  Affine and ArgMax are
// not defined by the reference; they are defined here
// with TypeOf descriptors in the reference's style (algebra.hpp:105-147).
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "forge/algebra.hpp"
#include "forge/primitives.hpp"
#include "../../include/forge.h"  // the repo C-ABI header, for the forge_op menu only

using namespace forge;
using namespace forge::prim;

namespace refd {

struct Affine {
  float a, b;
};
struct ArgMax {
  float v;
  int32_t i;
};

}  // namespace refd

namespace forge::intr {
template <>
struct TypeOf<refd::Affine> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::tuple(
        {TypeDescriptor::primitive(Scalar::F32), TypeDescriptor::primitive(Scalar::F32)});
    return d;
  }
};
template <>
struct TypeOf<refd::ArgMax> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::tuple(
        {TypeDescriptor::primitive(Scalar::F32), TypeDescriptor::primitive(Scalar::U32)});
    return d;
  }
};
}  // namespace forge::intr

namespace {

thread_local std::string g_err;

RunOptions make_opt(int backend, uint64_t seed) {
  RunOptions o;
  o.backend = backend == 1 ? Backend::Threads : Backend::Simulator;
  o.schedule.seed = seed;
  return o;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

template <class T, class S, class F, class Op>
int do_scan(const SemiringSpec<F, S, Op>& spec, const void* src, uint64_t n, void* dst,
            bool inclusive, int backend, uint64_t seed, double* wall) {
  Machine m;
  ArchParams p;
  BufferId a = intr::create_buffer<T>(m, n);
  BufferId b = intr::create_buffer<S>(m, n);
  if (n) m.write(a, std::span<const T>(static_cast<const T*>(src), n));
  Workspace ws = make_scan_workspace<S>(m, n, p);
  auto t0 = std::chrono::steady_clock::now();
  LaunchReport rep = scan(m, spec, intr::make_view<T>(m, a), intr::make_view<S>(m, b), inclusive,
                          ws, p, make_opt(backend, seed));
  double w = secs_since(t0);
  if (!rep.ok) {
    g_err = std::string("launch fault: ") + to_string(rep.fault.kind) + " " + rep.fault.detail;
    return 100;
  }
  if (n) m.read(b, std::span<S>(static_cast<S*>(dst), n));
  if (wall) *wall = backend == 1 && rep.wall_seconds > 0 ? rep.wall_seconds : w;
  return 0;
}

template <class T, class S, class F, class Op>
int do_mapreduce(const SemiringSpec<F, S, Op>& spec, const void* src, uint64_t n, void* out,
                 int backend, uint64_t seed, double* wall) {
  Machine m;
  ArchParams p;
  BufferId a = intr::create_buffer<T>(m, n);
  if (n) m.write(a, std::span<const T>(static_cast<const T*>(src), n));
  Workspace ws = make_mapreduce_workspace<S>(m, p);
  S r{};
  auto t0 = std::chrono::steady_clock::now();
  LaunchReport rep =
      mapreduce(m, spec, intr::make_view<T>(m, a), ws, p, &r, make_opt(backend, seed));
  double w = secs_since(t0);
  if (!rep.ok) {
    g_err = std::string("launch fault: ") + to_string(rep.fault.kind) + " " + rep.fault.detail;
    return 100;
  }
  std::memcpy(out, &r, sizeof(S));
  if (wall) *wall = backend == 1 && rep.wall_seconds > 0 ? rep.wall_seconds : w;
  return 0;
}

// matvec (which = 0), vecmat (which = 1); x == nullptr -> mapreduce_2d.
template <class T, class S, class F, class Op>
int do_mat(int which, const SemiringSpec<F, S, Op>& spec, const void* A, uint64_t n, uint64_t pc,
           const void* x, void* out, int backend, uint64_t seed, double* wall) {
  Machine m;
  ArchParams p;
  uint64_t outs = which == 0 ? pc : n;
  uint64_t red = which == 0 ? n : pc;
  BufferId a = intr::create_buffer<T>(m, n * pc);
  BufferId xb = intr::create_buffer<T>(m, red);
  BufferId yb = intr::create_buffer<S>(m, outs);
  if (n * pc) m.write(a, std::span<const T>(static_cast<const T*>(A), n * pc));
  if (x && red) m.write(xb, std::span<const T>(static_cast<const T*>(x), red));
  Workspace ws = make_mat_workspace<S>(m, red, outs, p);
  auto t0 = std::chrono::steady_clock::now();
  LaunchReport rep;
  RunOptions o = make_opt(backend, seed);
  if (which == 0)
    rep = matvec<T, S>(m, spec, intr::make_view<T>(m, a), n, pc, intr::make_view<T>(m, xb),
                       intr::make_view<S>(m, yb), ws, p, o, x != nullptr);
  else
    rep = vecmat<T, S>(m, spec, intr::make_view<T>(m, a), n, pc, intr::make_view<T>(m, xb),
                       intr::make_view<S>(m, yb), ws, p, o, x != nullptr);
  double w = secs_since(t0);
  if (!rep.ok) {
    g_err = std::string("launch fault: ") + to_string(rep.fault.kind) + " " + rep.fault.detail;
    return 100;
  }
  if (outs) m.read(yb, std::span<S>(static_cast<S*>(out), outs));
  if (wall) *wall = backend == 1 && rep.wall_seconds > 0 ? rep.wall_seconds : w;
  return 0;
}

constexpr float kInf = std::numeric_limits<float>::infinity();

// Visits the menu entry `op` with its SemiringSpec and (T, S).
template <class V>
int visit_1d(int op, V&& v) {
  auto id = [](auto x) { return x; };
  switch (op) {
    case FORGE_OP_F32_SUM:
      return v.template go<float>(make_semiring<float>(id, [](float a, float b) { return a + b; },
                                                       std::optional<float>(0.f), true));
    case FORGE_OP_F32_SUMSQ:
      return v.template go<float>(make_semiring<float>([](float x) { return x * x; },
                                                       [](float a, float b) { return a + b; },
                                                       std::optional<float>(0.f), true));
    case FORGE_OP_F32_MAX:
      return v.template go<float>(make_semiring<float>(
          id, [](float a, float b) { return a >= b ? a : b; }, std::optional<float>(-kInf), true));
    case FORGE_OP_F32_MIN:
      return v.template go<float>(make_semiring<float>(
          id, [](float a, float b) { return a <= b ? a : b; }, std::optional<float>(kInf), true));
    case FORGE_OP_F64_SUM:
      return v.template go<double>(make_semiring<double>(
          id, [](double a, double b) { return a + b; }, std::optional<double>(0.0), true));
    case FORGE_OP_I32_SUM:
      return v.template go<int32_t>(make_semiring<int32_t>(
          id, [](int32_t a, int32_t b) { return int32_t(uint32_t(a) + uint32_t(b)); },
          std::optional<int32_t>(0), true));
    case FORGE_OP_I32_MAX:
      return v.template go<int32_t>(make_semiring<int32_t>(
          id, [](int32_t a, int32_t b) { return a >= b ? a : b; },
          std::optional<int32_t>(std::numeric_limits<int32_t>::min()), true));
    case FORGE_OP_I32_MIN:
      return v.template go<int32_t>(make_semiring<int32_t>(
          id, [](int32_t a, int32_t b) { return a <= b ? a : b; },
          std::optional<int32_t>(std::numeric_limits<int32_t>::max()), true));
    case FORGE_OP_U32_SUM:
      return v.template go<uint32_t>(make_semiring<uint32_t>(
          id, [](uint32_t a, uint32_t b) { return a + b; }, std::optional<uint32_t>(0u), true));
    case FORGE_OP_I64_SUM:
      return v.template go<int64_t>(make_semiring<int64_t>(
          id, [](int64_t a, int64_t b) { return int64_t(uint64_t(a) + uint64_t(b)); },
          std::optional<int64_t>(0), true));
    case FORGE_OP_AFFINE_F32:
      return v.template go<refd::Affine>(make_semiring<refd::Affine>(
          id,
          [](refd::Affine p, refd::Affine q) { return refd::Affine{q.a * p.a, q.a * p.b + q.b}; },
          std::optional<refd::Affine>(refd::Affine{1.f, 0.f}), false));
    case FORGE_OP_ARGMAX_F32I32:
      return v.template go<refd::ArgMax>(make_semiring<refd::ArgMax>(
          id,
          [](refd::ArgMax a, refd::ArgMax b) {
            if (a.v > b.v) return a;
            if (b.v > a.v) return b;
            return a.i <= b.i ? a : b;
          },
          std::optional<refd::ArgMax>(
              refd::ArgMax{-kInf, std::numeric_limits<int32_t>::max()}),
          true));
    case FORGE_OP_MAT2_U32:
      return v.template go<alg::Mat2>(make_semiring<alg::Mat2>(
          id, [](const alg::Mat2& a, const alg::Mat2& b) { return alg::mat2_mul(a, b); },
          std::optional<alg::Mat2>(alg::mat2_one), false));
    case FORGE_OP_QUAT_F32:
      return v.template go<alg::Quaternion>(make_semiring<alg::Quaternion>(
          id,
          [](const alg::Quaternion& a, const alg::Quaternion& b) { return alg::qmul(a, b); },
          std::optional<alg::Quaternion>(alg::quat_one), false));
    case FORGE_OP_UF8_F32_SUM:
      return v.template go<alg::UnitFloat8>(make_semiring<float>(
          [](alg::UnitFloat8 c) { return alg::decode(c); },
          [](float a, float b) { return a + b; }, std::optional<float>(0.f), true));
    case FORGE_OP_F32_LOGSUMEXP:
      return v.template go<float>(make_semiring<float>(
          id, [](float a, float b) { return alg::log_sum_exp(a, b); },
          std::optional<float>(-kInf), true));
    default:
      g_err = "op not in the 1-D menu";
      return FORGE_ERR_UNSUPPORTED;
  }
}

template <class V>
int visit_2d(int op, V&& v) {
  switch (op) {
    case FORGE_OP_MV_F32_PLUS_TIMES:
      return v.template go<float>(make_semiring<float>([](float a, float b) { return a * b; },
                                                       [](float a, float b) { return a + b; },
                                                       std::optional<float>(0.f), true));
    case FORGE_OP_MV_F32_MIN_PLUS:
      return v.template go<float>(make_semiring<float>(
          [](float a, float b) { return a + b; }, [](float a, float b) { return a <= b ? a : b; },
          std::optional<float>(kInf), true));
    case FORGE_OP_MV_F32_MAX_PLUS:
      return v.template go<float>(make_semiring<float>(
          [](float a, float b) { return a + b; }, [](float a, float b) { return a >= b ? a : b; },
          std::optional<float>(-kInf), true));
    case FORGE_OP_MV_I32_PLUS_TIMES:
      return v.template go<int32_t>(make_semiring<int32_t>(
          [](int32_t a, int32_t b) { return int32_t(uint32_t(a) * uint32_t(b)); },
          [](int32_t a, int32_t b) { return int32_t(uint32_t(a) + uint32_t(b)); },
          std::optional<int32_t>(0), true));
    case FORGE_OP_MV_F64_PLUS_TIMES:
      return v.template go<double>(make_semiring<double>(
          [](double a, double b) { return a * b; }, [](double a, double b) { return a + b; },
          std::optional<double>(0.0), true));
    case FORGE_OP_MV_MAT2_U32:
      return v.template go<alg::Mat2>(make_semiring<alg::Mat2>(
          [](const alg::Mat2& a, const alg::Mat2& b) { return alg::mat2_mul(a, b); },
          [](const alg::Mat2& a, const alg::Mat2& b) { return alg::mat2_mul(a, b); },
          std::optional<alg::Mat2>(alg::mat2_one), false));
    default:
      g_err = "op not in the 2-D menu";
      return FORGE_ERR_UNSUPPORTED;
  }
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const forge::Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

}  // namespace


namespace {

struct ScanV {
  const void* src;
  uint64_t n;
  void* dst;
  bool incl;
  int backend;
  uint64_t seed;
  double* wall;
  template <class T, class Spec>
  int go(const Spec& spec) {
    using S = std::remove_cvref_t<decltype(*spec.identity)>;
    return do_scan<T, S>(spec, src, n, dst, incl, backend, seed, wall);
  }
};

struct MapReduceV {
  const void* src;
  uint64_t n;
  void* out;
  int backend;
  uint64_t seed;
  double* wall;
  template <class T, class Spec>
  int go(const Spec& spec) {
    using S = std::remove_cvref_t<decltype(*spec.identity)>;
    return do_mapreduce<T, S>(spec, src, n, out, backend, seed, wall);
  }
};

struct Mat2dV {
  int which;
  const void* A;
  uint64_t n, p;
  void* out;
  int backend;
  uint64_t seed;
  double* wall;
  template <class T, class Spec>
  int go(const Spec& spec) {
    using S = std::remove_cvref_t<decltype(*spec.identity)>;
    Machine m;
    ArchParams ap;
    BufferId a = intr::create_buffer<T>(m, n * p);
    uint64_t outs = which == 0 ? p : n;
    BufferId yb = intr::create_buffer<S>(m, outs);
    if (n * p) m.write(a, std::span<const T>(static_cast<const T*>(A), n * p));
    Workspace ws = make_mat_workspace<S>(m, which == 0 ? n : p, outs, ap);
    auto t0 = std::chrono::steady_clock::now();
    LaunchReport rep = mapreduce_2d<T, S>(m, spec, intr::make_view<T>(m, a), n, p,
                                          which == 0 ? ReduceAxis::Rows : ReduceAxis::Cols,
                                          intr::make_view<S>(m, yb), ws, ap,
                                          make_opt(backend, seed));
    double w = secs_since(t0);
    if (!rep.ok) {
      g_err = std::string("launch fault: ") + to_string(rep.fault.kind);
      return 100;
    }
    if (outs) m.read(yb, std::span<S>(static_cast<S*>(out), outs));
    if (wall) *wall = w;
    return 0;
  }
};

struct MatV {
  int which;
  const void* A;
  uint64_t n, p;
  const void* x;
  void* out;
  int backend;
  uint64_t seed;
  double* wall;
  template <class T, class Spec>
  int go(const Spec& spec) {
    using S = std::remove_cvref_t<decltype(*spec.identity)>;
    return do_mat<T, S>(which, spec, A, n, p, x, out, backend, seed, wall);
  }
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_scan(int op, int inclusive, const void* src, uint64_t n, void* dst, int backend,
             uint64_t seed, double* wall) {
  return guarded([&] {
    return visit_1d(op, ScanV{src, n, dst, inclusive != 0, backend, seed, wall});
  });
}

int ref_mapreduce(int op, const void* src, uint64_t n, void* out, int backend, uint64_t seed,
                  double* wall) {
  return guarded([&] { return visit_1d(op, MapReduceV{src, n, out, backend, seed, wall}); });
}

// which: 0 matvec, 1 vecmat.  x == NULL with a 1-D op runs mapreduce_2d
// (Rows for matvec, Cols for vecmat) through the reference's own delegation.
int ref_mat(int which, int op, const void* A, uint64_t n, uint64_t p, const void* x, void* out,
            int backend, uint64_t seed, double* wall) {
  if (x == nullptr)
    return guarded([&] { return visit_1d(op, Mat2dV{which, A, n, p, out, backend, seed, wall}); });
  return guarded([&] { return visit_2d(op, MatV{which, A, n, p, x, out, backend, seed, wall}); });
}

int ref_vcopy(const void* src, void* dst, uint64_t n, uint32_t elem_size, uint32_t nitem,
              int backend, double* wall) {
  return guarded([&]() -> int {
    Machine m;
    ArchParams p;
    TypeDescriptor d = elem_size == 1   ? TypeDescriptor::primitive(Scalar::U8)
                       : elem_size == 2 ? TypeDescriptor::primitive(Scalar::U16)
                       : elem_size == 8 ? TypeDescriptor::primitive(Scalar::U64)
                                        : TypeDescriptor::primitive(Scalar::U32);
    BufferId a = m.create_buffer(d, n), b = m.create_buffer(d, n);
    if (n) m.write_bytes(a, 0, std::span<const std::byte>((const std::byte*)src, n * elem_size));
    auto t0 = std::chrono::steady_clock::now();
    LaunchReport rep;
    if (elem_size == 4)
      rep = vcopy(m, intr::View<uint32_t>{a, 0, n, 1}, intr::View<uint32_t>{b, 0, n, 1}, nitem, p,
                  make_opt(backend, 0));
    else if (elem_size == 8)
      rep = vcopy(m, intr::View<uint64_t>{a, 0, n, 1}, intr::View<uint64_t>{b, 0, n, 1}, nitem,
                  p, make_opt(backend, 0));
    else if (elem_size == 2)
      rep = vcopy(m, intr::View<uint16_t>{a, 0, n, 1}, intr::View<uint16_t>{b, 0, n, 1}, nitem,
                  p, make_opt(backend, 0));
    else
      rep = vcopy(m, intr::View<uint8_t>{a, 0, n, 1}, intr::View<uint8_t>{b, 0, n, 1}, nitem, p,
                  make_opt(backend, 0));
    if (wall) *wall = secs_since(t0);
    if (!rep.ok) return 100;
    if (n) m.read_bytes(b, 0, std::span<std::byte>((std::byte*)dst, n * elem_size));
    return 0;
  });
}

int ref_vload_pattern(uint64_t offset, uint32_t nitem, uint32_t* segs, uint32_t* count) {
  return guarded([&] {
    intr::LoadPattern lp = intr::vload_pattern(offset, nitem);
    for (uint32_t i = 0; i < lp.count; ++i) segs[i] = lp.seg[i];
    *count = lp.count;
    return 0;
  });
}

int ref_required_workspace(int prim, uint32_t accum_size, uint64_t n, uint64_t p_cols,
                           uint64_t* out) {
  return guarded([&] {
    *out = required_workspace(static_cast<Primitive>(prim), accum_size, n, p_cols, ArchParams{});
    return 0;
  });
}

uint64_t ref_scan_tiles(uint64_t n) { return scan_tiles(n, ArchParams{}.normalized()); }

// Error-path probes (SURVEY.md §8(c) error KATs): exclusive scan without an
// identity, non-commutative mapreduce, empty mapreduce.  Returns the status.
int ref_error_probe(int which) {
  return guarded([&]() -> int {
    Machine m;
    ArchParams p;
    BufferId a = intr::create_buffer<int32_t>(m, 4);
    BufferId b = intr::create_buffer<int32_t>(m, 4);
    auto add = [](int32_t x, int32_t y) { return x + y; };
    auto id = [](int32_t x) { return x; };
    if (which == 0) {
      auto spec = make_semiring<int32_t>(id, add, std::nullopt, true);
      Workspace ws = make_scan_workspace<int32_t>(m, 4, p);
      scan(m, spec, intr::make_view<int32_t>(m, a), intr::make_view<int32_t>(m, b), false, ws, p);
    } else if (which == 1) {
      auto spec = make_semiring<int32_t>(id, add, std::optional<int32_t>(0), false);
      Workspace ws = make_mapreduce_workspace<int32_t>(m, p);
      int32_t r;
      mapreduce(m, spec, intr::make_view<int32_t>(m, a), ws, p, &r);
    } else if (which == 2) {
      auto spec = make_semiring<int32_t>(id, add, std::nullopt, true);
      Workspace ws = make_mapreduce_workspace<int32_t>(m, p);
      int32_t r;
      mapreduce(m, spec, intr::View<int32_t>{a, 0, 0, 1}, ws, p, &r);
    } else if (which == 3) {
      ArchParams bad;
      bad.warp_width = 48;
      bad.normalized();
    } else if (which == 4) {
      auto spec = make_semiring<int32_t>(id, add, std::optional<int32_t>(0), true);
      Workspace ws = make_scan_workspace<int32_t>(m, 4, p);
      scan(m, spec, intr::make_view<int32_t>(m, a), intr::View<int32_t>{b, 0, 3, 1}, true, ws, p);
    }
    return 0;
  });
}

}  // extern "C"
