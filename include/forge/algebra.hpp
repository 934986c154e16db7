// forge/algebra.hpp — element types and operator packages, host- and device-callable.
//
// Mirrors /root/reference/proj/include/forge/algebra.hpp:15-147 (UnitFloat8,
// Quaternion/qmul, Mat2/mat2_mul, MisalignedStruct, sat_add_i32, log_sum_exp
// and their TypeOf descriptors) with FORGE_HD (__host__ __device__) so the same
// functions run inside sm_100a kernels.  Adds the two BASELINE config-3 types
// the reference lacks:
//   Affine{a, b}: x -> a*x + b, compose(p, q) = "p then q" = {q.a*p.a, q.a*p.b + q.b}
//                 (associative, NOT commutative)
//   ArgMax{v, i}: max by v, ties to the smaller i (associative, commutative, exact)
// plus ready-made functor structs (Plus, Times, Min, Max, ...) usable as the
// `op` / `map` of a SemiringSpec in nvcc translation units.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>

#include "forge/intrinsics.hpp"

#ifndef FORGE_HD
#if defined(__CUDACC__)
#define FORGE_HD __host__ __device__ __forceinline__
#else
#define FORGE_HD inline
#endif
#endif

namespace forge::alg {

// ---- UnitFloat8: 256 levels on [-1, 1] (algebra.hpp:15-28)
struct UnitFloat8 {
  uint8_t code;
};

// decode = -1 + (2c)/255 with the quotient correctly rounded.  The IEEE division
// is replaced by a reciprocal multiply plus one FMA residual correction, which
// reproduces the correctly rounded quotient for every one of the 256 codes
// (checked exhaustively: tests/test_capi_cpu.py, tests/test_gpu_primitives.py)
// at a fraction of the cost of a full-range division on the GPU.
FORGE_HD float decode(UnitFloat8 v) {
  const float x = 2.0f * float(v.code);
  const float r = 1.0f / 255.0f;
#if defined(__CUDA_ARCH__)
  const float q = __fmul_rn(x, r);
  const float res = __fmaf_rn(-q, 255.0f, x);
  const float t = __fmaf_rn(res, r, q);
  return __fadd_rn(-1.0f, t);
#else
  const float q = x * r;
  const float res = std::fma(-q, 255.0f, x);
  const float t = std::fma(res, r, q);
  return -1.0f + t;
#endif
}

FORGE_HD UnitFloat8 encode(float x) {
  if (x <= -1.0f) return {0};
  if (x >= 1.0f) return {255};
  const float scaled = (x + 1.0f) * 0.5f * 255.0f;
#if defined(__CUDA_ARCH__)
  return {static_cast<uint8_t>(rintf(scaled))};
#else
  return {static_cast<uint8_t>(std::nearbyint(scaled))};
#endif
}

// ---- Quaternions, Hamilton product (algebra.hpp:33-46)
struct Quaternion {
  float w, x, y, z;
};

FORGE_HD Quaternion qmul(const Quaternion& a, const Quaternion& b) {
  return Quaternion{
      a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z,
      a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
      a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
      a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w,
  };
}

inline constexpr Quaternion quat_one{1.0f, 0.0f, 0.0f, 0.0f};

// ---- 2x2 wrapping-u32 matrices (algebra.hpp:52-69): exact, non-commutative
struct Mat2 {
  uint32_t m[4];  // row-major
};

FORGE_HD Mat2 mat2_mul(const Mat2& a, const Mat2& b) {
  Mat2 r;
  r.m[0] = a.m[0] * b.m[0] + a.m[1] * b.m[2];
  r.m[1] = a.m[0] * b.m[1] + a.m[1] * b.m[3];
  r.m[2] = a.m[2] * b.m[0] + a.m[3] * b.m[2];
  r.m[3] = a.m[2] * b.m[1] + a.m[3] * b.m[3];
  return r;
}

inline constexpr Mat2 mat2_one{{1, 0, 0, 1}};

FORGE_HD bool operator==(const Mat2& a, const Mat2& b) {
  return a.m[0] == b.m[0] && a.m[1] == b.m[1] && a.m[2] == b.m[2] && a.m[3] == b.m[3];
}

// ---- padding test type (algebra.hpp:75-80): byte@0, double@8, short@16, size 24
struct MisalignedStruct {
  int8_t a;
  double b;
  int16_t c;
};
static_assert(sizeof(MisalignedStruct) == 24);

// ---- affine maps and arg-max (new for BASELINE config 3)
template <class F>
struct AffineT {
  F a, b;
};
using Affine = AffineT<float>;

template <class F>
FORGE_HD AffineT<F> affine_compose(const AffineT<F>& p, const AffineT<F>& q) {
  return AffineT<F>{q.a * p.a, q.a * p.b + q.b};
}

// ---- order-independent f32 max / min.  The reference's
// `a >= b ? a : b` is neither commutative on ±0 nor associative with NaN, so
// a GPU tree and a sequential fold could disagree bit-wise on such inputs.
// Here: any NaN operand gives the canonical NaN 0x7fffffff (the PTX canonical
// NaN, so the device needs no fix-up); -0 < +0 (max(-0, +0) = +0,
// min(-0, +0) = -0).  On ordinary values it equals the reference operator.
// Device: one FMNMX.NAN instruction (max.NaN / min.NaN).
FORGE_HD bool is_nan_f32(float x) { return x != x; }
FORGE_HD uint32_t f32_bits(float x) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(x);
#else
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
#endif
}
FORGE_HD float f32_from_bits(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float x;
  std::memcpy(&x, &u, 4);
  return x;
#endif
}
inline constexpr uint32_t kCanonicalNaN32 = 0x7fffffffu;

FORGE_HD float fmax_total(float a, float b) {
#if defined(__CUDA_ARCH__)
  // FMNMX.NAN: NaN -> 0x7fffffff, and -0 < +0 in either operand order
  // (measured on B200, tools/probe_minmax.cu) — exactly the semantics above
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
#else
  if (is_nan_f32(a) || is_nan_f32(b)) return f32_from_bits(kCanonicalNaN32);
  if (a == b) return std::signbit(a) ? b : a;  // equal: differ at most in the sign of zero
  return a > b ? a : b;
#endif
}
FORGE_HD float fmin_total(float a, float b) {
#if defined(__CUDA_ARCH__)
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
#else
  if (is_nan_f32(a) || is_nan_f32(b)) return f32_from_bits(kCanonicalNaN32);
  if (a == b) return std::signbit(a) ? a : b;
  return a < b ? a : b;
#endif
}

struct ArgMax {
  float v;
  int32_t i;
};

// max by v, ties to the smaller i.  NaN values rank above every number (the
// arg-max of data containing NaN is its first NaN); -0 == +0 ties by index.
// A total preorder on v, so the op is associative and commutative for every
// input, NaN included.  (Branch-free selects: as cheap as the NaN-unaware form.)
// sa / sb: a / b strictly better.  !(x <= y) is "x > y or unordered" (one
// FSETP.GTU): with the other side's NaN masked off it is exactly "x > y, or x
// NaN and y not" — 4 FSETP per combine instead of 5.
FORGE_HD ArgMax argmax_combine(const ArgMax& a, const ArgMax& b) {
  const bool an = is_nan_f32(a.v), bn = is_nan_f32(b.v);
  const bool sa = !(a.v <= b.v) & !bn;
  const bool sb = !(b.v <= a.v) & !an;
  return (sa | (!sb & (a.i <= b.i))) ? a : b;
}

// ---- operator helpers (algebra.hpp:85-100)
FORGE_HD int32_t sat_add_i32(int32_t a, int32_t b) {
  const int64_t s = int64_t(a) + int64_t(b);
  if (s > int64_t(INT32_MAX)) return INT32_MAX;
  if (s < int64_t(INT32_MIN)) return INT32_MIN;
  return int32_t(s);
}

namespace detail {
FORGE_HD float lse_log1p(float x) {
#if defined(__CUDA_ARCH__)
  return log1pf(x);
#else
  return std::log1p(x);
#endif
}
FORGE_HD double lse_log1p(double x) {
#if defined(__CUDA_ARCH__)
  return ::log1p(x);
#else
  return std::log1p(x);
#endif
}
FORGE_HD float lse_exp(float x) {
#if defined(__CUDA_ARCH__)
  return expf(x);
#else
  return std::exp(x);
#endif
}
FORGE_HD double lse_exp(double x) {
#if defined(__CUDA_ARCH__)
  return ::exp(x);
#else
  return std::exp(x);
#endif
}
template <class F>
FORGE_HD bool neg_inf(F v) {
  return v == -std::numeric_limits<F>::infinity();
}
}  // namespace detail

// op(a, b) = log(exp a + exp b), identity -inf.
template <class F>
FORGE_HD F log_sum_exp(F a, F b) {
  if (detail::neg_inf(a)) return b;
  if (detail::neg_inf(b)) return a;
  const F hi = a > b ? a : b;
  const F lo = a > b ? b : a;
  return hi + detail::lse_log1p(detail::lse_exp(lo - hi));
}

// ---------------------------------------------------------------------------
// Functor structs (usable as SemiringSpec map/op in nvcc translation units).

struct Identity {
  template <class T>
  FORGE_HD T operator()(const T& x) const { return x; }
};
struct Square {
  template <class T>
  FORGE_HD T operator()(const T& x) const { return x * x; }
};
struct Plus {
  template <class T>
  FORGE_HD T operator()(const T& a, const T& b) const { return a + b; }
};
struct Times {
  template <class T>
  FORGE_HD T operator()(const T& a, const T& b) const { return a * b; }
};
struct Min {
  template <class T>
  FORGE_HD T operator()(const T& a, const T& b) const { return a <= b ? a : b; }
};
struct Max {
  template <class T>
  FORGE_HD T operator()(const T& a, const T& b) const { return a >= b ? a : b; }
};
struct WrapPlusI32 {
  FORGE_HD int32_t operator()(int32_t a, int32_t b) const { return int32_t(uint32_t(a) + uint32_t(b)); }
};
struct WrapTimesI32 {
  FORGE_HD int32_t operator()(int32_t a, int32_t b) const { return int32_t(uint32_t(a) * uint32_t(b)); }
};
struct WrapPlusI64 {
  FORGE_HD int64_t operator()(int64_t a, int64_t b) const { return int64_t(uint64_t(a) + uint64_t(b)); }
};
struct QMul {
  FORGE_HD Quaternion operator()(const Quaternion& a, const Quaternion& b) const { return qmul(a, b); }
};
struct Mat2Mul {
  FORGE_HD Mat2 operator()(const Mat2& a, const Mat2& b) const { return mat2_mul(a, b); }
};
struct AffineCompose {
  FORGE_HD Affine operator()(const Affine& p, const Affine& q) const { return affine_compose(p, q); }
};
struct ArgMaxOp {
  FORGE_HD ArgMax operator()(const ArgMax& a, const ArgMax& b) const { return argmax_combine(a, b); }
};
struct LogSumExp {
  template <class F>
  FORGE_HD F operator()(F a, F b) const { return log_sum_exp(a, b); }
};
struct DecodeUF8 {
  // decode is affine in the code: -1 + (2/255) c.  Mapreduce with a real sum
  // may fold the codes exactly as integers (forge/cuda/reduce.cuh code sums).
  static constexpr bool kAffineCode = true;
  static constexpr double kCodeOffset = -1.0;
  static constexpr double kCodeScale = 2.0 / 255.0;
  FORGE_HD float operator()(UnitFloat8 c) const { return decode(c); }
};

}  // namespace forge::alg

namespace forge::intr {

template <>
struct TypeOf<alg::UnitFloat8> : detail::ScalarTypeOf<Scalar::U8> {};

namespace detail {
inline TypeDescriptor tuple_of(Scalar s, int n) {
  std::vector<TypeDescriptor> e;
  for (int i = 0; i < n; ++i) e.push_back(TypeDescriptor::primitive(s));
  return TypeDescriptor::tuple(std::move(e));
}
}  // namespace detail

template <>
struct TypeOf<alg::Quaternion> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::F32, 4);
    return d;
  }
};
template <>
struct TypeOf<alg::Mat2> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::U32, 4);
    return d;
  }
};
template <>
struct TypeOf<alg::Affine> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = detail::tuple_of(Scalar::F32, 2);
    return d;
  }
};
template <>
struct TypeOf<alg::ArgMax> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::tuple(
        {TypeDescriptor::primitive(Scalar::F32), TypeDescriptor::primitive(Scalar::U32)});
    return d;
  }
};
template <>
struct TypeOf<alg::MisalignedStruct> {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::struct_of(
        {{TypeDescriptor::primitive(Scalar::U8), 0},
         {TypeDescriptor::primitive(Scalar::F64), 8},
         {TypeDescriptor::primitive(Scalar::U16), 16}},
        sizeof(alg::MisalignedStruct));
    return d;
  }
};

}  // namespace forge::intr
