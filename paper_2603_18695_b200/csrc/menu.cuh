// menu.cuh — the fixed operator menu of the C-ABI (include/forge.h forge_op).
//
// Each entry binds (T, S, map, op, identity, commutative) like a SemiringSpec
// (primitives.hpp:92-104).  The f32 / f64 / affine / quaternion / log-sum-exp
// ops carry their inter-tile chains in double precision (CarryTraits,
// forge/cuda/reduce.cuh); per-element work stays in S.
#pragma once

#include <cfloat>
#include <climits>
#include <cmath>

#include "forge.h"
#include "forge/algebra.hpp"
#include "forge/primitives.hpp"

namespace forge::menu {

using namespace forge::alg;

#ifndef FORGE_AFFINE_NARROW_EMIT
#define FORGE_AFFINE_NARROW_EMIT 1
#endif

// ---- carry policies
struct F32SumCarry {
  using C = double;
  static constexpr bool kWide = false;  // sums: f32 per element, f64 across tiles
  static __device__ __forceinline__ C to_c(float s) { return double(s); }
  static __device__ __forceinline__ float to_s(C c) { return float(c); }
  template <class Op>
  static __device__ __forceinline__ C op(const Op&, C a, C b) { return a + b; }
};

struct AffineCarry {
  using C = AffineT<double>;
  static constexpr bool kWide = true;        // product chain: aggregates and carries in f64 ...
  static constexpr bool kNarrowEmit = FORGE_AFFINE_NARROW_EMIT;  // ... per-row output prefixes in f32
  static __device__ __forceinline__ C to_c(const Affine& s) { return C{double(s.a), double(s.b)}; }
  static __device__ __forceinline__ Affine to_s(const C& c) { return Affine{float(c.a), float(c.b)}; }
  template <class Op>
  static __device__ __forceinline__ C op(const Op&, const C& p, const C& q) { return affine_compose(p, q); }
};

struct QuatD {
  double w, x, y, z;
};
struct QuatCarry {
  using C = QuatD;
  static constexpr bool kWide = true;  // product chain: whole scan in f64
  static __device__ __forceinline__ C to_c(const Quaternion& q) { return C{q.w, q.x, q.y, q.z}; }
  static __device__ __forceinline__ Quaternion to_s(const C& c) {
    return Quaternion{float(c.w), float(c.x), float(c.y), float(c.z)};
  }
  template <class Op>
  static __device__ __forceinline__ C op(const Op&, const C& a, const C& b) {
    return C{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
             a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
  }
};

struct LseCarry {
  using C = double;
  static constexpr bool kWide = false;
  static __device__ __forceinline__ C to_c(float s) { return double(s); }
  static __device__ __forceinline__ float to_s(C c) { return float(c); }
  template <class Op>
  static __device__ __forceinline__ C op(const Op&, C a, C b) { return log_sum_exp(a, b); }
};

// ---- operators
struct AddF32 {
  using carry_traits = F32SumCarry;
  static constexpr bool kRealSum = true;  // a real-number sum (code sums may fold exactly)
  FORGE_HD float operator()(float a, float b) const { return a + b; }
};
struct AddF64 {
  FORGE_HD double operator()(double a, double b) const { return a + b; }
};
struct MaxF32 {  // NaN -> canonical NaN, -0 < +0: order-independent (algebra.hpp)
  FORGE_HD float operator()(float a, float b) const { return fmax_total(a, b); }
};
struct MinF32 {
  FORGE_HD float operator()(float a, float b) const { return fmin_total(a, b); }
};
struct MaxI32 {
  FORGE_HD int32_t operator()(int32_t a, int32_t b) const { return a >= b ? a : b; }
};
struct MinI32 {
  FORGE_HD int32_t operator()(int32_t a, int32_t b) const { return a <= b ? a : b; }
};
struct AddU32 {
  FORGE_HD uint32_t operator()(uint32_t a, uint32_t b) const { return a + b; }
};
struct AffineOp {
  using carry_traits = AffineCarry;
  FORGE_HD Affine operator()(const Affine& p, const Affine& q) const { return affine_compose(p, q); }
};
struct QuatOp {
  using carry_traits = QuatCarry;
  FORGE_HD Quaternion operator()(const Quaternion& a, const Quaternion& b) const { return qmul(a, b); }
};
struct LseOp {
  using carry_traits = LseCarry;
  FORGE_HD float operator()(float a, float b) const { return log_sum_exp(a, b); }
};
struct MulF32 {
  FORGE_HD float operator()(float a, float b) const { return a * b; }
};
struct AddF32Map {  // f(a, b) = a + b for the tropical semirings (no carry policy needed)
  FORGE_HD float operator()(float a, float b) const { return a + b; }
};
struct MulF64 {
  FORGE_HD double operator()(double a, double b) const { return a * b; }
};

// ---- entries
template <class T_, class S_, class F_, class Op_>
struct Entry {
  using T = T_;
  using S = S_;
  using F = F_;
  using Op = Op_;
  S identity;
  bool commutative;
  forge_op op;
  const char* name;

  prim::SemiringSpec<F, S, Op> spec(bool with_identity) const {
    return prim::SemiringSpec<F, S, Op>{F{}, Op{}, with_identity ? std::optional<S>(identity) : std::nullopt,
                                        commutative};
  }
};

constexpr float kInfF = __builtin_huge_valf();

// Calls v(entry) with the 1-D menu entry for `op`; returns FORGE_ERR_UNSUPPORTED otherwise.
template <class V>
int visit1(forge_op op, V&& v) {
  switch (op) {
    case FORGE_OP_F32_SUM: return v(Entry<float, float, Identity, AddF32>{0.f, true, op, "f32_sum"});
    case FORGE_OP_F32_SUMSQ: return v(Entry<float, float, Square, AddF32>{0.f, true, op, "f32_sumsq"});
    case FORGE_OP_F32_MAX: return v(Entry<float, float, Identity, MaxF32>{-kInfF, true, op, "f32_max"});
    case FORGE_OP_F32_MIN: return v(Entry<float, float, Identity, MinF32>{kInfF, true, op, "f32_min"});
    case FORGE_OP_F64_SUM: return v(Entry<double, double, Identity, AddF64>{0.0, true, op, "f64_sum"});
    case FORGE_OP_I32_SUM: return v(Entry<int32_t, int32_t, Identity, WrapPlusI32>{0, true, op, "i32_sum"});
    case FORGE_OP_I32_MAX: return v(Entry<int32_t, int32_t, Identity, MaxI32>{INT32_MIN, true, op, "i32_max"});
    case FORGE_OP_I32_MIN: return v(Entry<int32_t, int32_t, Identity, MinI32>{INT32_MAX, true, op, "i32_min"});
    case FORGE_OP_U32_SUM: return v(Entry<uint32_t, uint32_t, Identity, AddU32>{0u, true, op, "u32_sum"});
    case FORGE_OP_I64_SUM: return v(Entry<int64_t, int64_t, Identity, WrapPlusI64>{0, true, op, "i64_sum"});
    case FORGE_OP_AFFINE_F32:
      return v(Entry<Affine, Affine, Identity, AffineOp>{Affine{1.f, 0.f}, false, op, "affine_f32"});
    case FORGE_OP_ARGMAX_F32I32:
      return v(Entry<ArgMax, ArgMax, Identity, ArgMaxOp>{ArgMax{-kInfF, INT32_MAX}, true, op, "argmax_f32i32"});
    case FORGE_OP_MAT2_U32: return v(Entry<Mat2, Mat2, Identity, Mat2Mul>{mat2_one, false, op, "mat2_u32"});
    case FORGE_OP_QUAT_F32: return v(Entry<Quaternion, Quaternion, Identity, QuatOp>{quat_one, false, op, "quat_f32"});
    case FORGE_OP_UF8_F32_SUM: return v(Entry<UnitFloat8, float, DecodeUF8, AddF32>{0.f, true, op, "uf8_f32_sum"});
    case FORGE_OP_F32_LOGSUMEXP: return v(Entry<float, float, Identity, LseOp>{-kInfF, true, op, "f32_logsumexp"});
    default: return FORGE_ERR_UNSUPPORTED;
  }
}

template <class V>
int visit2(forge_op op, V&& v) {
  switch (op) {
    case FORGE_OP_MV_F32_PLUS_TIMES: return v(Entry<float, float, MulF32, AddF32>{0.f, true, op, "mv_f32_plus_times"});
    case FORGE_OP_MV_F32_MIN_PLUS: return v(Entry<float, float, AddF32Map, MinF32>{kInfF, true, op, "mv_f32_min_plus"});
    case FORGE_OP_MV_F32_MAX_PLUS: return v(Entry<float, float, AddF32Map, MaxF32>{-kInfF, true, op, "mv_f32_max_plus"});
    case FORGE_OP_MV_I32_PLUS_TIMES:
      return v(Entry<int32_t, int32_t, WrapTimesI32, WrapPlusI32>{0, true, op, "mv_i32_plus_times"});
    case FORGE_OP_MV_F64_PLUS_TIMES: return v(Entry<double, double, MulF64, AddF64>{0.0, true, op, "mv_f64_plus_times"});
    case FORGE_OP_MV_MAT2_U32: return v(Entry<Mat2, Mat2, Mat2Mul, Mat2Mul>{mat2_one, false, op, "mv_mat2_u32"});
    default: return FORGE_ERR_UNSUPPORTED;
  }
}

}  // namespace forge::menu
