// test_templates.cu — the C++ drop-in API used the way a reference user would:
// user-defined element types and operators (functor structs and
// __host__ __device__ lambdas) through forge/primitives.hpp, checked against
// plain sequential folds on the host.  Built by __graft_entry__.build()
// (Makefile target `cpptests`), run by tests/test_gpu_cpp.py on a B200.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "forge/algebra.hpp"
#include "forge/primitives.hpp"

using namespace forge;
using prim::ArchParams;
using prim::make_semiring;

namespace {

int g_fail = 0, g_pass = 0;

#define EXPECT(cond, ...)                  \
  do {                                     \
    if (cond) {                            \
      ++g_pass;                            \
    } else {                               \
      ++g_fail;                            \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);            \
      std::printf("\n");                   \
    }                                      \
  } while (0)

// ---- user types (not in the menu) ----------------------------------------
struct Mat3 {  // 3x3 wrapping-u32 matrices: exact, non-commutative
  uint32_t m[9];
};
struct Mat3Mul {
  FORGE_HD Mat3 operator()(const Mat3& a, const Mat3& b) const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        uint32_t s = 0;
        for (int k = 0; k < 3; ++k) s += a.m[3 * i + k] * b.m[3 * k + j];
        r.m[3 * i + j] = s;
      }
    return r;
  }
};
bool eq(const Mat3& a, const Mat3& b) { return std::memcmp(&a, &b, sizeof(Mat3)) == 0; }

struct MinMax {  // (min, max) pair: exact, commutative
  float lo, hi;
};

struct Tri {  // 12-byte struct: not a power-of-two size (scalar paths)
  int32_t a, b, c;
};
struct TriAdd {
  FORGE_HD Tri operator()(const Tri& x, const Tri& y) const {
    return Tri{int32_t(uint32_t(x.a) + uint32_t(y.a)), int32_t(uint32_t(x.b) + uint32_t(y.b)),
               int32_t(uint32_t(x.c) ^ uint32_t(y.c))};
  }
};

}  // namespace

namespace forge::intr {
template <>
struct TypeOf<Mat3> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::U32, 9);
    return d;
  }
};
template <>
struct TypeOf<MinMax> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::F32, 2);
    return d;
  }
};
template <>
struct TypeOf<Tri> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::U32, 3);
    return d;
  }
};
}  // namespace forge::intr

namespace {

template <class T>
BufferId upload(Machine& m, const std::vector<T>& v) {
  BufferId b = intr::create_buffer<T>(m, v.size());
  if (!v.empty()) m.write(b, std::span<const T>(v));
  return b;
}

template <class T>
std::vector<T> download(Machine& m, BufferId b, uint64_t n) {
  std::vector<T> v(n);
  if (n) m.read(b, std::span<T>(v));
  return v;
}

void test_scan_mat3(Machine& m) {
  std::mt19937 rng(7);
  for (uint64_t n : {1ull, 31ull, 257ull, 4097ull, 100003ull, 1000003ull}) {
    std::vector<Mat3> x(n);
    for (auto& v : x)
      for (auto& e : v.m) e = rng();
    auto spec = make_semiring<Mat3>(alg::Identity{}, Mat3Mul{}, std::optional<Mat3>(Mat3{{1, 0, 0, 0, 1, 0, 0, 0, 1}}),
                                    false);
    ArchParams p;
    BufferId a = upload(m, x), d = intr::create_buffer<Mat3>(m, n);
    prim::Workspace ws = prim::make_scan_workspace<Mat3>(m, n, p);
    for (bool incl : {true, false}) {
      LaunchReport rep = prim::scan(m, spec, intr::make_view<Mat3>(m, a), intr::make_view<Mat3>(m, d), incl, ws, p);
      auto got = download<Mat3>(m, d, n);
      Mat3 acc = Mat3{{1, 0, 0, 0, 1, 0, 0, 0, 1}};
      bool ok = rep.ok;
      for (uint64_t i = 0; i < n && ok; ++i) {
        if (!incl) ok = eq(got[i], acc);
        acc = Mat3Mul{}(acc, x[i]);
        if (incl) ok = ok && eq(got[i], acc);
      }
      EXPECT(ok, "scan Mat3 n=%llu incl=%d", (unsigned long long)n, int(incl));
    }
    ws.release(m);
    m.destroy_buffer(a);
    m.destroy_buffer(d);
  }
}

void test_mapreduce_lambda(Machine& m) {
  std::mt19937 rng(11);
  std::uniform_real_distribution<float> U(-100.f, 100.f);
  const uint64_t n = 3000017;
  std::vector<float> x(n);
  for (auto& v : x) v = U(rng);
  auto f = [] __host__ __device__(float v) { return MinMax{v, v}; };
  auto op = [] __host__ __device__(MinMax a, MinMax b) {
    return MinMax{a.lo < b.lo ? a.lo : b.lo, a.hi > b.hi ? a.hi : b.hi};
  };
  auto spec = make_semiring<MinMax>(f, op, std::optional<MinMax>(), true);
  ArchParams p;
  BufferId a = upload(m, x);
  prim::Workspace ws = prim::make_mapreduce_workspace<MinMax>(m, p);
  MinMax r{};
  LaunchReport rep = prim::mapreduce(m, spec, intr::make_view<float>(m, a), ws, p, &r);
  float lo = x[0], hi = x[0];
  for (float v : x) lo = v < lo ? v : lo, hi = v > hi ? v : hi;
  EXPECT(rep.ok && r.lo == lo && r.hi == hi, "mapreduce MinMax lambda: got (%g,%g) want (%g,%g)", r.lo, r.hi, lo, hi);
  EXPECT(rep.wall_seconds > 0, "wall_seconds is the CUDA-event time");
  // strided view (every 3rd element from offset 2)
  intr::View<float> v3 = intr::make_view<float>(m, a).strided(2, (n - 2 + 2) / 3, 3);
  rep = prim::mapreduce(m, spec, v3, ws, p, &r);
  lo = x[2], hi = x[2];
  for (uint64_t i = 2; i < n; i += 3) lo = x[i] < lo ? x[i] : lo, hi = x[i] > hi ? x[i] : hi;
  EXPECT(rep.ok && r.lo == lo && r.hi == hi, "mapreduce strided view");
  // empty input: identity required
  try {
    prim::mapreduce(m, spec, intr::View<float>{a, 0, 0, 1}, ws, p, &r);
    EXPECT(false, "empty mapreduce without identity must raise");
  } catch (const Error& e) {
    EXPECT(e.code() == ErrorCode::MissingIdentity, "MissingIdentity");
  }
  ws.release(m);
  m.destroy_buffer(a);
}

void test_tri_scan_scalar_path(Machine& m) {
  const uint64_t n = 50001;
  std::vector<Tri> x(n);
  std::mt19937 rng(5);
  for (auto& v : x) v = Tri{int32_t(rng()), int32_t(rng()), int32_t(rng())};
  auto spec = make_semiring<Tri>(alg::Identity{}, TriAdd{}, std::optional<Tri>(Tri{0, 0, 0}), true);
  ArchParams p;
  BufferId a = upload(m, x), d = intr::create_buffer<Tri>(m, n);
  prim::Workspace ws = prim::make_scan_workspace<Tri>(m, n, p);
  LaunchReport rep = prim::scan(m, spec, intr::make_view<Tri>(m, a), intr::make_view<Tri>(m, d), true, ws, p);
  auto got = download<Tri>(m, d, n);
  Tri acc{0, 0, 0};
  bool ok = rep.ok;
  for (uint64_t i = 0; i < n && ok; ++i) {
    acc = TriAdd{}(acc, x[i]);
    ok = std::memcmp(&acc, &got[i], sizeof(Tri)) == 0;
  }
  EXPECT(ok, "scan of a 12-byte struct");
  // mapreduce over the same (commutative: + and xor)
  prim::Workspace wm = prim::make_mapreduce_workspace<Tri>(m, p);
  Tri r{};
  rep = prim::mapreduce(m, spec, intr::make_view<Tri>(m, a), wm, p, &r);
  EXPECT(rep.ok && std::memcmp(&r, &acc, sizeof(Tri)) == 0, "mapreduce of a 12-byte struct");
  ws.release(m);
  wm.release(m);
}

void test_matrix_custom_semiring(Machine& m) {
  // bottleneck semiring: f = min(x, a), op = max (exact, commutative)
  auto f2 = [] __host__ __device__(int32_t u, int32_t v) { return u < v ? u : v; };
  auto opmax = [] __host__ __device__(int32_t u, int32_t v) { return u > v ? u : v; };
  auto spec = make_semiring<int32_t>(f2, opmax, std::optional<int32_t>(INT32_MIN), true);
  std::mt19937 rng(3);
  for (auto [n, pc] : {std::pair<uint64_t, uint64_t>{1000, 300}, {3, 7}, {4096, 64}, {65, 1000}}) {
    std::vector<int32_t> A(n * pc), xm(n), xv(pc);
    for (auto& v : A) v = int32_t(rng() % 100000);
    for (auto& v : xm) v = int32_t(rng() % 100000);
    for (auto& v : xv) v = int32_t(rng() % 100000);
    ArchParams p;
    BufferId ab = upload(m, A), xb = upload(m, xm), xvb = upload(m, xv);
    BufferId yb = intr::create_buffer<int32_t>(m, pc), zb = intr::create_buffer<int32_t>(m, n);
    prim::Workspace ws = prim::make_mat_workspace<int32_t>(m, n, pc, p);
    LaunchReport r1 = prim::matvec<int32_t, int32_t>(m, spec, intr::make_view<int32_t>(m, ab), n, pc,
                                                     intr::make_view<int32_t>(m, xb), intr::make_view<int32_t>(m, yb), ws, p);
    LaunchReport r2 = prim::vecmat<int32_t, int32_t>(m, spec, intr::make_view<int32_t>(m, ab), n, pc,
                                                     intr::make_view<int32_t>(m, xvb), intr::make_view<int32_t>(m, zb), ws, p);
    auto y = download<int32_t>(m, yb, pc), z = download<int32_t>(m, zb, n);
    bool ok = r1.ok && r2.ok;
    for (uint64_t j = 0; j < pc && ok; ++j) {
      int32_t acc = INT32_MIN;
      for (uint64_t i = 0; i < n; ++i) acc = opmax(acc, f2(xm[i], A[j * n + i]));
      ok = y[j] == acc;
    }
    for (uint64_t i = 0; i < n && ok; ++i) {
      int32_t acc = INT32_MIN;
      for (uint64_t j = 0; j < pc; ++j) acc = opmax(acc, f2(A[j * n + i], xv[j]));
      ok = z[i] == acc;
    }
    EXPECT(ok, "bottleneck-semiring matvec/vecmat %llux%llu", (unsigned long long)n, (unsigned long long)pc);
    // mapreduce_2d: column / row sums (wrapping)
    auto sum = make_semiring<int32_t>(alg::Identity{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
    prim::mapreduce_2d<int32_t, int32_t>(m, sum, intr::make_view<int32_t>(m, ab), n, pc, prim::ReduceAxis::Rows,
                                         intr::make_view<int32_t>(m, yb), ws, p);
    prim::mapreduce_2d<int32_t, int32_t>(m, sum, intr::make_view<int32_t>(m, ab), n, pc, prim::ReduceAxis::Cols,
                                         intr::make_view<int32_t>(m, zb), ws, p);
    y = download<int32_t>(m, yb, pc);
    z = download<int32_t>(m, zb, n);
    ok = true;
    for (uint64_t j = 0; j < pc && ok; ++j) {
      uint32_t s = 0;
      for (uint64_t i = 0; i < n; ++i) s += uint32_t(A[j * n + i]);
      ok = uint32_t(y[j]) == s;
    }
    for (uint64_t i = 0; i < n && ok; ++i) {
      uint32_t s = 0;
      for (uint64_t j = 0; j < pc; ++j) s += uint32_t(A[j * n + i]);
      ok = uint32_t(z[i]) == s;
    }
    EXPECT(ok, "mapreduce_2d rows/cols %llux%llu", (unsigned long long)n, (unsigned long long)pc);
    ws.release(m);
  }
}

void test_noncommutative_matvec(Machine& m) {
  // Mat2 semiring: ordered path must keep row order exactly.
  const uint64_t n = 3000, pc = 20;
  std::vector<alg::Mat2> A(n * pc), x(n);
  std::mt19937 rng(9);
  for (auto& v : A)
    for (auto& e : v.m) e = rng();
  for (auto& v : x)
    for (auto& e : v.m) e = rng();
  auto spec = make_semiring<alg::Mat2>(alg::Mat2Mul{}, alg::Mat2Mul{}, std::optional<alg::Mat2>(alg::mat2_one), false);
  ArchParams p;
  BufferId ab = upload(m, A), xb = upload(m, x), yb = intr::create_buffer<alg::Mat2>(m, pc);
  prim::Workspace ws = prim::make_mat_workspace<alg::Mat2>(m, n, pc, p);
  LaunchReport r = prim::matvec<alg::Mat2, alg::Mat2>(m, spec, intr::make_view<alg::Mat2>(m, ab), n, pc,
                                                      intr::make_view<alg::Mat2>(m, xb), intr::make_view<alg::Mat2>(m, yb), ws, p);
  auto y = download<alg::Mat2>(m, yb, pc);
  bool ok = r.ok;
  for (uint64_t j = 0; j < pc && ok; ++j) {
    alg::Mat2 acc = alg::mat2_one;
    for (uint64_t i = 0; i < n; ++i) acc = alg::mat2_mul(acc, alg::mat2_mul(x[i], A[j * n + i]));
    ok = acc == y[j];
  }
  EXPECT(ok, "non-commutative Mat2 matvec keeps row order");
}

void test_errors_and_params(Machine& m) {
  ArchParams p;
  BufferId a = intr::create_buffer<int32_t>(m, 16), b = intr::create_buffer<int32_t>(m, 8);
  auto spec_noid = make_semiring<int32_t>(alg::Identity{}, alg::WrapPlusI32{}, std::optional<int32_t>(), true);
  prim::Workspace ws = prim::make_scan_workspace<int32_t>(m, 16, p);
  auto expect_code = [&](auto&& fn, ErrorCode c, const char* what) {
    try {
      fn();
      EXPECT(false, "%s: no error", what);
    } catch (const Error& e) {
      EXPECT(e.code() == c, "%s: got %s", what, to_string(e.code()));
    }
  };
  expect_code([&] { prim::scan(m, spec_noid, intr::make_view<int32_t>(m, a), intr::make_view<int32_t>(m, a), false, ws, p); },
              ErrorCode::MissingIdentity, "exclusive scan without identity");
  expect_code([&] { prim::scan(m, spec_noid, intr::make_view<int32_t>(m, a), intr::make_view<int32_t>(m, b), true, ws, p); },
              ErrorCode::DimensionMismatch, "scan length mismatch");
  auto nc = make_semiring<int32_t>(alg::Identity{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), false);
  prim::Workspace wm = prim::make_mapreduce_workspace<int32_t>(m, p);
  int32_t r;
  expect_code([&] { prim::mapreduce(m, nc, intr::make_view<int32_t>(m, a), wm, p, &r); }, ErrorCode::InvalidArgument,
              "non-commutative mapreduce");
  ArchParams w64;
  w64.warp_width = 64;
  expect_code([&] { (void)w64.normalized(); }, ErrorCode::Unsupported, "warp_width 64");
  ArchParams bad;
  bad.nitem_scan = 3;
  expect_code([&] { (void)bad.normalized(); }, ErrorCode::InvalidNitem, "nitem 3");
  expect_code([&] { (void)intr::make_view<double>(m, a); }, ErrorCode::InvalidArgument, "view element size");
  BufferId big = intr::create_buffer<int32_t>(m, 1 << 20), bigd = intr::create_buffer<int32_t>(m, 1 << 20);
  auto ok = make_semiring<int32_t>(alg::Identity{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
  expect_code([&] { prim::scan(m, ok, intr::make_view<int32_t>(m, big), intr::make_view<int32_t>(m, bigd), true, ws, p); },
              ErrorCode::WorkspaceTooSmall, "scan workspace too small");
  // validate_reduce_op (primitives.hpp:108-118)
  std::mt19937 rng(1);
  bool assoc = prim::validate_reduce_op<alg::Mat2>(alg::Mat2Mul{}, std::optional<alg::Mat2>(alg::mat2_one), false,
                                                   [&] { return alg::Mat2{{uint32_t(rng()), uint32_t(rng()), uint32_t(rng()), uint32_t(rng())}}; },
                                                   [](const alg::Mat2& u, const alg::Mat2& v) { return u == v; });
  bool comm = prim::validate_reduce_op<alg::Mat2>(alg::Mat2Mul{}, std::optional<alg::Mat2>(alg::mat2_one), true,
                                                  [&] { return alg::Mat2{{uint32_t(rng()), uint32_t(rng()), uint32_t(rng()), uint32_t(rng())}}; },
                                                  [](const alg::Mat2& u, const alg::Mat2& v) { return u == v; });
  EXPECT(assoc && !comm, "validate_reduce_op: Mat2 associative, not commutative");
}

void test_vcopy_struct(Machine& m) {
  const uint64_t n = 10007;
  std::vector<alg::MisalignedStruct> x(n);
  for (uint64_t i = 0; i < n; ++i) x[i] = alg::MisalignedStruct{int8_t(i), double(i) * 0.5, int16_t(i * 3)};
  BufferId a = upload(m, x), b = intr::create_buffer<alg::MisalignedStruct>(m, n);
  ArchParams p;
  LaunchReport r = prim::vcopy(m, intr::make_view<alg::MisalignedStruct>(m, a), intr::make_view<alg::MisalignedStruct>(m, b), 4, p);
  auto y = download<alg::MisalignedStruct>(m, b, n);
  bool ok = r.ok;
  const auto& d = intr::descriptor_of<alg::MisalignedStruct>();
  for (uint64_t i = 0; i < n && ok; ++i)
    ok = value_bytes_equal(d, std::as_bytes(std::span(&x[i], 1)), std::as_bytes(std::span(&y[i], 1)));
  EXPECT(ok, "vcopy of MisalignedStruct");
  EXPECT(r.buffers.size() == m.buffer_count() && r.buffers[a].load_elems == n && r.buffers[b].store_elems == n,
         "LaunchReport counters: one load and one store per element");
}


// ---- mixed-width map paths (algebra.hpp:15-28): u8 / u16 / i8
// inputs promoted by the map to f32 / i32, through mapreduce and scan; plus a
// 16-byte T scanned into a 4-byte S through make_scan_workspace<S> (a
// workspace sized for S must fit every T: ADVICE r01).
struct Half {  // u8 -> f32: x / 2 (exact)
  FORGE_HD float operator()(uint8_t c) const { return 0.5f * float(c); }
};
// A map affine in the code plus a real-number sum: mapreduce takes the exact
// integer code-sum path (IDP4A, forge/cuda/reduce.cuh) for these.
struct Centered {  // u8 -> f32: (c - 127.5) / 4
  static constexpr bool kAffineCode = true;
  static constexpr double kCodeOffset = -127.5 / 4.0;
  static constexpr double kCodeScale = 0.25;
  FORGE_HD float operator()(uint8_t c) const { return 0.25f * (float(c) - 127.5f); }
};
struct RealPlusF32 {
  static constexpr bool kRealSum = true;
  FORGE_HD float operator()(float a, float b) const { return a + b; }
};
struct Widen16 {  // u16 -> i32
  FORGE_HD int32_t operator()(uint16_t c) const { return int32_t(c); }
};
struct SignedByte {  // i8 -> i32
  FORGE_HD int32_t operator()(int8_t c) const { return int32_t(c); }
};
struct Quad {
  uint32_t w[4];
};
struct QuadSum {  // 16-byte T -> 4-byte S (wrapping sum of the words)
  FORGE_HD uint32_t operator()(const Quad& q) const { return q.w[0] + q.w[1] + q.w[2] + q.w[3]; }
};
}  // namespace
namespace forge::intr {
template <>
struct TypeOf<Quad> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::U32, 4);
    return d;
  }
};
}  // namespace forge::intr
namespace {

void test_mixed_width_maps(Machine& m) {
  std::mt19937 rng(21);
  ArchParams p;
  for (uint64_t n : {1ull, 33ull, 4097ull, 1000003ull, 5000011ull}) {
    std::vector<uint8_t> x8(n);
    std::vector<uint16_t> x16(n);
    std::vector<int8_t> xs8(n);
    for (uint64_t i = 0; i < n; ++i) {
      x8[i] = uint8_t(rng());
      x16[i] = uint16_t(rng());
      xs8[i] = int8_t(rng());
    }
    BufferId b8 = upload(m, x8), b16 = upload(m, x16), bs8 = upload(m, xs8);
    // u8 -> f32 sum: floating point, the SURVEY §8(c) rule |got - exact| <= 1e-5 * sum|terms|
    auto s_half = make_semiring<float>(Half{}, alg::Plus{}, std::optional<float>(0.f), true);
    prim::Workspace wf = prim::make_mapreduce_workspace<float>(m, p);
    float rf = 0;
    LaunchReport r = prim::mapreduce(m, s_half, intr::make_view<uint8_t>(m, b8), wf, p, &rf);
    double want = 0;
    for (uint8_t c : x8) want += 0.5 * c;
    EXPECT(r.ok && std::abs(double(rf) - want) <= 1e-5 * want, "u8->f32 mapreduce n=%llu: %.9g vs %.9g",
           (unsigned long long)n, rf, want);
    // exact code sums (affine map + real sum), aligned and misaligned (head/tail bytes) views
    auto s_c = make_semiring<float>(Centered{}, RealPlusF32{}, std::optional<float>(0.f), true);
    for (uint64_t off : {0ull, 3ull}) {
      if (off >= n) continue;
      float rc = 0;
      r = prim::mapreduce(m, s_c, intr::make_view<uint8_t>(m, b8).strided(off, n - off, 1), wf, p, &rc);
      double ex = 0, sc = 0;
      for (uint64_t i = off; i < n; ++i) ex += 0.25 * (double(x8[i]) - 127.5), sc += std::abs(0.25 * (double(x8[i]) - 127.5));
      EXPECT(r.ok && std::abs(double(rc) - ex) <= 1e-5 * sc + 1e-30, "u8 code-sum mapreduce n=%llu off=%llu: %.9g vs %.9g",
             (unsigned long long)n, (unsigned long long)off, rc, ex);
    }
    // u16 -> i32 wrapping sum, u16 max
    auto s_w = make_semiring<int32_t>(Widen16{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
    prim::Workspace wi = prim::make_mapreduce_workspace<int32_t>(m, p);
    int32_t ri = 0;
    r = prim::mapreduce(m, s_w, intr::make_view<uint16_t>(m, b16), wi, p, &ri);
    uint32_t wsum = 0;
    for (uint16_t c : x16) wsum += c;
    EXPECT(r.ok && uint32_t(ri) == wsum, "u16->i32 mapreduce n=%llu", (unsigned long long)n);
    // i8 -> i32 inclusive scan (exact), and u8 -> f32 exclusive scan
    auto s_sb = make_semiring<int32_t>(SignedByte{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
    BufferId d32 = intr::create_buffer<int32_t>(m, n), df = intr::create_buffer<float>(m, n);
    prim::Workspace ws = prim::make_scan_workspace<int32_t>(m, n, p);
    r = prim::scan(m, s_sb, intr::make_view<int8_t>(m, bs8), intr::make_view<int32_t>(m, d32), true, ws, p);
    auto g32 = download<int32_t>(m, d32, n);
    bool ok = r.ok;
    int32_t acc = 0;
    for (uint64_t i = 0; i < n && ok; ++i) ok = g32[i] == (acc += xs8[i]);
    EXPECT(ok, "i8->i32 scan n=%llu", (unsigned long long)n);
    prim::Workspace wsf = prim::make_scan_workspace<float>(m, n, p);
    r = prim::scan(m, s_half, intr::make_view<uint8_t>(m, b8), intr::make_view<float>(m, df), false, wsf, p);
    auto gf = download<float>(m, df, n);
    ok = r.ok;
    double accf = 0;
    for (uint64_t i = 0; i < n && ok; ++i) {
      ok = std::abs(double(gf[i]) - accf) <= 1e-5 * accf;  // terms are >= 0: sum|terms| = the prefix
      accf += 0.5 * x8[i];
    }
    EXPECT(ok, "u8->f32 exclusive scan n=%llu", (unsigned long long)n);
    // 16-byte T -> 4-byte S scan with the S-sized workspace
    std::vector<Quad> q(n);
    for (auto& v : q)
      for (auto& w : v.w) w = rng();
    BufferId bq = upload(m, q);
    auto s_q = make_semiring<uint32_t>(QuadSum{}, alg::Plus{}, std::optional<uint32_t>(0u), true);
    prim::Workspace wq = prim::make_scan_workspace<uint32_t>(m, n, p);
    BufferId du = intr::create_buffer<uint32_t>(m, n);
    r = prim::scan(m, s_q, intr::make_view<Quad>(m, bq), intr::make_view<uint32_t>(m, du), true, wq, p);
    auto gu = download<uint32_t>(m, du, n);
    ok = r.ok;
    uint32_t accu = 0;
    for (uint64_t i = 0; i < n && ok; ++i) ok = gu[i] == (accu += QuadSum{}(q[i]));
    EXPECT(ok, "16-byte T -> 4-byte S scan through make_scan_workspace<S> n=%llu", (unsigned long long)n);
    for (BufferId b : {b8, b16, bs8, d32, df, bq, du}) m.destroy_buffer(b);
    for (prim::Workspace* w : {&wf, &wi, &ws, &wsf, &wq}) w->release(m);
  }
}

// ---- one workspace buffer serving several primitives and matrix shapes in
// turn (layouts overlap; the library re-zeroes on a layout change)
void test_workspace_shared_across_primitives(Machine& m) {
  ArchParams p;
  std::mt19937 rng(33);
  const uint64_t nt = 200003, pt = 8;   // tall-skinny: gevm splits rows (tickets + partials)
  const uint64_t nw = 1000, pw = 60000; // short-wide: gemv splits columns
  std::vector<int32_t> At(nt * pt), xt(nt), Aw(nw * pw), xw(pw), v(nt);
  for (auto& e : At) e = int32_t(rng() % 1000);
  for (auto& e : xt) e = int32_t(rng() % 1000);
  for (auto& e : Aw) e = int32_t(rng() % 1000);
  for (auto& e : xw) e = int32_t(rng() % 1000);
  for (auto& e : v) e = int32_t(rng());
  auto pt_spec = make_semiring<int32_t>(alg::WrapTimesI32{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
  auto sum = make_semiring<int32_t>(alg::Identity{}, alg::WrapPlusI32{}, std::optional<int32_t>(0), true);
  BufferId bAt = upload(m, At), bxt = upload(m, xt), bAw = upload(m, Aw), bxw = upload(m, xw), bv = upload(m, v);
  BufferId y = intr::create_buffer<int32_t>(m, pt), z = intr::create_buffer<int32_t>(m, nw);
  BufferId sd = intr::create_buffer<int32_t>(m, nt);
  // one byte buffer big enough for every layout, wired into every field
  const uint64_t big = std::max({prim::required_workspace(prim::Primitive::MatVec, 4, nt, pt, p),
                                 prim::required_workspace(prim::Primitive::VecMat, 4, nw, pw, p),
                                 prim::required_workspace(prim::Primitive::Scan, 4, nt, 0, p),
                                 prim::required_workspace(prim::Primitive::MapReduce, 4, nt, 0, p)});
  prim::Workspace ws;
  ws.partials = ws.tile_flag = intr::create_buffer<uint8_t>(m, big, 256);
  ws.result = intr::create_buffer<uint8_t>(m, 64, 256);
  std::vector<uint32_t> wy(pt, 0), wz(nw, 0);
  for (uint64_t j = 0; j < pt; ++j)
    for (uint64_t i = 0; i < nt; ++i) wy[j] += uint32_t(xt[i]) * uint32_t(At[j * nt + i]);
  for (uint64_t i = 0; i < nw; ++i)
    for (uint64_t j = 0; j < pw; ++j) wz[i] += uint32_t(Aw[j * nw + i]) * uint32_t(xw[j]);
  uint32_t wsum = 0;
  for (int32_t e : v) wsum += uint32_t(e);
  bool ok = true;
  for (int round = 0; round < 3; ++round) {
    prim::matvec<int32_t, int32_t>(m, pt_spec, intr::make_view<int32_t>(m, bAt), nt, pt, intr::make_view<int32_t>(m, bxt),
                                   intr::make_view<int32_t>(m, y), ws, p);
    auto gy = download<int32_t>(m, y, pt);
    for (uint64_t j = 0; j < pt; ++j) ok = ok && uint32_t(gy[j]) == wy[j];
    prim::scan(m, sum, intr::make_view<int32_t>(m, bv), intr::make_view<int32_t>(m, sd), true, ws, p);
    auto gs = download<int32_t>(m, sd, nt);
    uint32_t acc = 0;
    for (uint64_t i = 0; i < nt; ++i) ok = ok && uint32_t(gs[i]) == (acc += uint32_t(v[i]));
    prim::vecmat<int32_t, int32_t>(m, pt_spec, intr::make_view<int32_t>(m, bAw), nw, pw, intr::make_view<int32_t>(m, bxw),
                                   intr::make_view<int32_t>(m, z), ws, p);
    auto gz = download<int32_t>(m, z, nw);
    for (uint64_t i = 0; i < nw; ++i) ok = ok && uint32_t(gz[i]) == wz[i];
    int32_t r = 0;
    prim::mapreduce(m, sum, intr::make_view<int32_t>(m, bv), ws, p, &r);
    ok = ok && uint32_t(r) == wsum;
  }
  EXPECT(ok, "one workspace buffer shared by matvec / scan / vecmat / mapreduce, 3 rounds");
  for (BufferId b : {bAt, bxt, bAw, bxw, bv, y, z, sd, ws.partials, ws.result}) m.destroy_buffer(b);
}

// ---- reference API re-exports: MatPlan / tall_slices / plan_mat
// (primitives.hpp:202-244) with the reference's own numbers,
// TypeOf<OptVal<S>> (:840-853), sat_add_i32 (algebra.hpp:85-90)
void test_reference_api_reexports(Machine& m) {
  ArchParams p;
  prim::MatPlan w = prim::plan_mat(16384, 16384, true, p);
  EXPECT(w.wide && w.cfg.num_blocks == 200 && w.cfg.threads_per_block == 128,
         "plan_mat C4 commutative: wide 200x128 (got wide=%d %ux%u)", int(w.wide), w.cfg.num_blocks,
         w.cfg.threads_per_block);
  prim::MatPlan t = prim::plan_mat(16384, 16384, false, p);
  EXPECT(!t.wide && t.nb == 2 && t.cfg.num_blocks == 400 && t.cfg.threads_per_block == 256 && t.slots == 2 * 16384,
         "plan_mat C4 non-commutative: tall nb=2 400x256");
  EXPECT(prim::tall_slices(1, p) == 1 && prim::tall_slices(8192, p) == 1 && prim::tall_slices(8193, p) == 2 &&
             prim::tall_slices(uint64_t(1) << 40, p) == 100,
         "tall_slices clamps to [1, mapreduce_blocks]");
  prim::MatPlan b = prim::b200_plan_mat<float>(prim::Primitive::MatVec, 16384, 16384, true);
  prim::MatPlan bv = prim::b200_plan_mat<float>(prim::Primitive::VecMat, 16384, 16384, true);
  EXPECT(b.wide && b.cfg.num_blocks > 0 && bv.nb >= 1 && bv.cfg.num_blocks > 0, "b200_plan_mat geometry");
  EXPECT(intr::descriptor_of<prim::OptVal<float>>() == parse_descriptor("struct(f32@0,u8@4;size=8)"),
         "TypeOf<OptVal<f32>> = %s", to_string(intr::descriptor_of<prim::OptVal<float>>()).c_str());
  EXPECT(intr::descriptor_of<prim::OptVal<alg::Mat2>>() ==
             parse_descriptor("struct(tuple(u32,u32,u32,u32)@0,u8@16;size=20)"),
         "TypeOf<OptVal<Mat2>> = %s", to_string(intr::descriptor_of<prim::OptVal<alg::Mat2>>()).c_str());
  // sat_add_i32 saturates, so it is NOT associative near the limits: the
  // reference's validate_reduce_op must reject it there and accept it on
  // small values (where it is plain addition)
  std::mt19937 rng(4);
  auto eqi = [](int32_t a, int32_t b) { return a == b; };
  auto sat = [](int32_t a, int32_t b) { return alg::sat_add_i32(a, b); };
  const bool big = prim::validate_reduce_op<int32_t>(sat, std::optional<int32_t>(0), true,
                                                     [&] { return int32_t(rng()); }, eqi);
  const bool small = prim::validate_reduce_op<int32_t>(sat, std::optional<int32_t>(0), true,
                                                       [&] { return int32_t(rng() % 1000) - 500; }, eqi);
  EXPECT(!big && small, "sat_add_i32: validate_reduce_op rejects saturation, accepts small values");
  EXPECT(alg::sat_add_i32(INT32_MAX, 1) == INT32_MAX && alg::sat_add_i32(INT32_MIN, -1) == INT32_MIN &&
             alg::sat_add_i32(2, 3) == 5,
         "sat_add_i32 known answers");
  // ... and on the device, as a mapreduce over values that never saturate
  std::vector<int32_t> x(100003);
  int64_t want = 0;
  for (auto& e : x) want += (e = int32_t(rng() % 20001) - 10000);
  BufferId bx = upload(m, x);
  auto spec = make_semiring<int32_t>(alg::Identity{}, [] __host__ __device__(int32_t a, int32_t c) {
    return alg::sat_add_i32(a, c);
  }, std::optional<int32_t>(0), true);
  prim::Workspace wm = prim::make_mapreduce_workspace<int32_t>(m, p);
  int32_t r = 0;
  LaunchReport rep = prim::mapreduce(m, spec, intr::make_view<int32_t>(m, bx), wm, p, &r);
  EXPECT(rep.ok && int64_t(r) == want, "sat_add_i32 mapreduce on the device");
  wm.release(m);
  m.destroy_buffer(bx);
}

}  // namespace

int main() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    std::printf("no CUDA device\n");
    return 2;
  }
  Machine m;
  test_scan_mat3(m);
  test_mapreduce_lambda(m);
  test_tri_scan_scalar_path(m);
  test_matrix_custom_semiring(m);
  test_noncommutative_matvec(m);
  test_errors_and_params(m);
  test_vcopy_struct(m);
  test_mixed_width_maps(m);
  test_workspace_shared_across_primitives(m);
  test_reference_api_reexports(m);
  std::printf("%s: %d passed, %d failed\n", g_fail ? "FAIL" : "PASS", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
