/*
 * oracle.c — sequential CPU restatement of the reference primitives.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): never linked into libforge.so and
 * never called by the product path.  Semantics follow
 *   mapreduce      /root/reference/proj/include/forge/primitives.hpp:348-431
 *   scan           primitives.hpp:440-603 (exclusive output rule :587-595)
 *   matvec/vecmat  primitives.hpp:775-807 (column-major A, f argument order)
 *   mapreduce_2d   primitives.hpp:814-836
 *   vload_pattern  intrinsics.hpp:198-211, intrinsics.cpp:29-33
 *   operator types algebra.hpp:15-100
 * Exact operators fold sequentially in S (any fold order of an associative op
 * gives the same value, so a left fold IS the reference result).  Floating
 * operators apply the map f in S precision (as the reference does) and fold
 * in 64-bit (long double for f64 data), returning the exact value plus the
 * error scale sum |terms| used by the tolerance rule of SURVEY.md §8(c).
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* generator                                                                 */

uint64_t orc_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static float gen_f32_sym(uint64_t u) { /* [-1, 1) on the exact grid k * 2^-23 */
  return (float)(int32_t)(u >> 40) * 0x1p-23f - 1.0f;
}
static float gen_f32_pos(uint64_t u) { /* [0, 1) on the grid k * 2^-24 */
  return (float)(int32_t)(u >> 40) * 0x1p-24f;
}

float orc_uf8_decode(uint8_t code) { /* algebra.hpp:19 */
  float t = 2.0f * (float)code;
  t = t / 255.0f;
  return -1.0f + t;
}

uint8_t orc_uf8_encode(float x) { /* algebra.hpp:22-28: nearest, ties to even */
  if (x <= -1.0f) return 0;
  if (x >= 1.0f) return 255;
  float scaled = (x + 1.0f) * 0.5f * 255.0f;
  return (uint8_t)nearbyintf(scaled);
}

/* variant 2 of the f32 ops: special values for the order-independence tests
 * of max / min / argmax (about 1 in 2^15 elements a NaN with a random payload
 * and sign, 1 in 2^15 an infinity, 1/8 a signed zero, 1/16 a small integer,
 * the rest gen_f32_sym).  Mirrored bit for bit by capi.cu's fill_kernel. */
static float gen_f32_special(uint64_t u) {
  const uint32_t low = (uint32_t)(u & 0xFFFFu);
  uint32_t bits;
  float f;
  if (low < 2u) {
    bits = 0x7fc00000u | (uint32_t)((u >> 16) & 0x3FFFFFu) | (low ? 0x80000000u : 0u);
  } else if (low < 4u) {
    bits = low == 2u ? 0x7f800000u : 0xff800000u;
  } else if (low < 0x2000u) {
    bits = (u >> 16) & 1u ? 0x80000000u : 0u;
  } else if (low < 0x3000u) {
    f = (float)(int32_t)((u >> 16) & 7u) - 4.0f;
    return f;
  } else {
    return gen_f32_sym(u);
  }
  memcpy(&f, &bits, 4);
  return f;
}

static void gen_one(forge_op op, uint64_t u, uint64_t idx, int32_t variant, unsigned char* out) {
  switch (op) {
    case FORGE_OP_F32_SUM:
    case FORGE_OP_F32_SUMSQ:
    case FORGE_OP_F32_MAX:
    case FORGE_OP_F32_MIN:
    case FORGE_OP_F32_LOGSUMEXP:
    case FORGE_OP_MV_F32_PLUS_TIMES:
    case FORGE_OP_MV_F32_MIN_PLUS:
    case FORGE_OP_MV_F32_MAX_PLUS: {
      float v = variant == 1 ? gen_f32_pos(u) : variant == 2 ? gen_f32_special(u) : gen_f32_sym(u);
      memcpy(out, &v, 4);
      break;
    }
    case FORGE_OP_F64_SUM:
    case FORGE_OP_MV_F64_PLUS_TIMES: {
      double v = (double)(int64_t)(u >> 11) * 0x1p-52 - 1.0;
      memcpy(out, &v, 8);
      break;
    }
    case FORGE_OP_I32_SUM:
    case FORGE_OP_I32_MAX:
    case FORGE_OP_I32_MIN:
    case FORGE_OP_U32_SUM:
    case FORGE_OP_MV_I32_PLUS_TIMES: {
      uint32_t v = (uint32_t)(u >> 32);
      if (variant == 1) v &= 0xFFu; /* small values: no wrap in sums */
      memcpy(out, &v, 4);
      break;
    }
    case FORGE_OP_I64_SUM: {
      memcpy(out, &u, 8);
      break;
    }
    case FORGE_OP_AFFINE_F32: {
      forge_affine_f32 v;
      v.a = 1.0f + (float)((int32_t)((u >> 50) & 0x3FFF) - 8192) * 0x1p-23f;
      v.b = (float)(int32_t)((u >> 8) & 0xFFFFFF) * 0x1p-23f - 1.0f;
      memcpy(out, &v, 8);
      break;
    }
    case FORGE_OP_ARGMAX_F32I32: {
      forge_argmax v;
      v.v = variant == 1 ? (float)(int32_t)((u >> 60) & 0xF) : variant == 2 ? gen_f32_special(u) : gen_f32_sym(u);
      v.i = (int32_t)(uint32_t)idx;
      memcpy(out, &v, 8);
      break;
    }
    case FORGE_OP_MAT2_U32:
    case FORGE_OP_MV_MAT2_U32: {
      uint64_t u2 = orc_mix(u);
      forge_mat2_u32 v;
      /* odd diagonal, even off-diagonal: det is odd, so every prefix product
         stays invertible mod 2^32 (uniform entries make long products collapse
         to the zero matrix, and scans of them test nothing past the first
         few hundred elements) */
      v.m[0] = (uint32_t)u | 1u;
      v.m[1] = (uint32_t)(u >> 32) & ~1u;
      v.m[2] = (uint32_t)u2 & ~1u;
      v.m[3] = (uint32_t)(u2 >> 32) | 1u;
      memcpy(out, &v, 16);
      break;
    }
    case FORGE_OP_QUAT_F32: {
      /* unit quaternions; explicit single roundings so host and device agree */
      uint64_t u2 = orc_mix(u);
      volatile float w = gen_f32_sym(u), x = gen_f32_sym(u << 24), y = gen_f32_sym(u2),
                     z = gen_f32_sym(u2 << 24);
      volatile float ww = w * w, xx = x * x, yy = y * y, zz = z * z;
      volatile float s1 = ww + xx, s2 = s1 + yy, s3 = s2 + zz;
      float r = sqrtf(s3 > 0x1p-20f ? s3 : 1.0f);
      forge_quat_f32 v = {w / r, x / r, y / r, z / r};
      memcpy(out, &v, 16);
      break;
    }
    case FORGE_OP_UF8_F32_SUM: {
      *out = (unsigned char)(u >> 56);
      break;
    }
    default:
      break;
  }
}

static uint32_t t_size_of(forge_op op) {
  switch (op) {
    case FORGE_OP_F64_SUM:
    case FORGE_OP_I64_SUM:
    case FORGE_OP_AFFINE_F32:
    case FORGE_OP_ARGMAX_F32I32:
    case FORGE_OP_MV_F64_PLUS_TIMES:
      return 8;
    case FORGE_OP_MAT2_U32:
    case FORGE_OP_QUAT_F32:
    case FORGE_OP_MV_MAT2_U32:
      return 16;
    case FORGE_OP_UF8_F32_SUM:
      return 1;
    default:
      return 4;
  }
}

static uint32_t s_size_of(forge_op op) {
  if (op == FORGE_OP_UF8_F32_SUM) return 4;
  return t_size_of(op);
}

int orc_fill_synthetic(forge_op op, void* dst, uint64_t n, uint64_t seed, uint64_t index_base,
                       int32_t variant) {
  uint32_t ts = t_size_of(op);
  unsigned char* p = (unsigned char*)dst;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t idx = index_base + i;
    gen_one(op, orc_mix(seed ^ idx), idx, variant, p + i * ts);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* operator algebra                                                          */

int orc_float_components(forge_op op) {
  switch (op) {
    case FORGE_OP_F32_SUM:
    case FORGE_OP_F32_SUMSQ:
    case FORGE_OP_F64_SUM:
    case FORGE_OP_UF8_F32_SUM:
    case FORGE_OP_F32_LOGSUMEXP:
    case FORGE_OP_MV_F32_PLUS_TIMES:
    case FORGE_OP_MV_F64_PLUS_TIMES:
      return 1;
    case FORGE_OP_AFFINE_F32:
      return 2;
    case FORGE_OP_QUAT_F32:
      return 4;
    default:
      return 0;
  }
}

/* Exact S values (16 bytes covers every menu S). */
typedef union sval {
  float f;
  double d;
  int32_t i;
  uint32_t u;
  int64_t l;
  forge_affine_f32 af;
  forge_argmax am;
  forge_mat2_u32 m2;
  forge_quat_f32 q;
  unsigned char raw[16];
} sval;

static forge_mat2_u32 mat2_mul(forge_mat2_u32 a, forge_mat2_u32 b) { /* algebra.hpp:56-63 */
  forge_mat2_u32 r;
  r.m[0] = a.m[0] * b.m[0] + a.m[1] * b.m[2];
  r.m[1] = a.m[0] * b.m[1] + a.m[1] * b.m[3];
  r.m[2] = a.m[2] * b.m[0] + a.m[3] * b.m[2];
  r.m[3] = a.m[2] * b.m[1] + a.m[3] * b.m[3];
  return r;
}

/* Order-independent f32 max / min (include/forge/algebra.hpp fmax_total):
 * NaN -> the canonical NaN 0x7fffffff (PTX's), -0 < +0.  Equal to the reference's
 * `a >= b ? a : b` (algebra ops of SPEC.md) on NaN-free inputs without
 * zero-sign ties, where that operator is itself order-dependent. */
static float canonical_nan(void) {
  const uint32_t bits = 0x7fffffffu;
  float f;
  memcpy(&f, &bits, 4);
  return f;
}
static float fmax_total(float a, float b) {
  if (a != a || b != b) return canonical_nan();
  if (a == b) return signbit(a) ? b : a;
  return a > b ? a : b;
}
static float fmin_total(float a, float b) {
  if (a != a || b != b) return canonical_nan();
  if (a == b) return signbit(a) ? a : b;
  return a < b ? a : b;
}

/* ArgMax (new BASELINE C3 type): max by v, ties to the smaller i; NaN ranks
 * above every number, so the op stays associative with NaN inputs. */
static forge_argmax argmax_op(forge_argmax a, forge_argmax b) {
  const int an = a.v != a.v, bn = b.v != b.v;
  if (an != bn) return an ? a : b;
  if (!an) {
    if (a.v > b.v) return a;
    if (b.v > a.v) return b;
  }
  return a.i <= b.i ? a : b;
}

static sval identity_of(forge_op op) {
  sval s;
  memset(&s, 0, sizeof s);
  switch (op) {
    case FORGE_OP_F32_MAX:
    case FORGE_OP_F32_LOGSUMEXP:
    case FORGE_OP_MV_F32_MAX_PLUS:
      s.f = -INFINITY;
      break;
    case FORGE_OP_F32_MIN:
    case FORGE_OP_MV_F32_MIN_PLUS:
      s.f = INFINITY;
      break;
    case FORGE_OP_I32_MAX:
      s.i = INT32_MIN;
      break;
    case FORGE_OP_I32_MIN:
      s.i = INT32_MAX;
      break;
    case FORGE_OP_AFFINE_F32:
      s.af.a = 1.0f;
      s.af.b = 0.0f;
      break;
    case FORGE_OP_ARGMAX_F32I32:
      s.am.v = -INFINITY;
      s.am.i = INT32_MAX;
      break;
    case FORGE_OP_MAT2_U32:
    case FORGE_OP_MV_MAT2_U32:
      s.m2.m[0] = 1;
      s.m2.m[3] = 1;
      break;
    case FORGE_OP_QUAT_F32:
      s.q.w = 1.0f;
      break;
    default:
      break;
  }
  return s;
}

/* f: T -> S for the exact 1-D ops (primitives.hpp:389, the map is applied per element). */
static sval map_exact(forge_op op, const unsigned char* t) {
  sval s;
  memset(&s, 0, sizeof s);
  memcpy(s.raw, t, t_size_of(op));
  return s;
}

/* a op b for exact ops (op order: a is the older / left operand). */
static sval combine_exact(forge_op op, sval a, sval b) {
  sval r;
  memset(&r, 0, sizeof r);
  switch (op) {
    case FORGE_OP_F32_MAX:
    case FORGE_OP_MV_F32_MAX_PLUS:
      r.f = fmax_total(a.f, b.f);
      break;
    case FORGE_OP_F32_MIN:
    case FORGE_OP_MV_F32_MIN_PLUS:
      r.f = fmin_total(a.f, b.f);
      break;
    case FORGE_OP_I32_SUM:
    case FORGE_OP_U32_SUM:
    case FORGE_OP_MV_I32_PLUS_TIMES:
      r.u = a.u + b.u;
      break;
    case FORGE_OP_I32_MAX:
      r.i = a.i >= b.i ? a.i : b.i;
      break;
    case FORGE_OP_I32_MIN:
      r.i = a.i <= b.i ? a.i : b.i;
      break;
    case FORGE_OP_I64_SUM:
      r.l = (int64_t)((uint64_t)a.l + (uint64_t)b.l);
      break;
    case FORGE_OP_ARGMAX_F32I32:
      r.am = argmax_op(a.am, b.am);
      break;
    case FORGE_OP_MAT2_U32:
    case FORGE_OP_MV_MAT2_U32:
      r.m2 = mat2_mul(a.m2, b.m2);
      break;
    default:
      break;
  }
  return r;
}

/* Float ops: exact accumulators in long double. */
typedef struct facc {
  long double v[4];     /* exact value components */
  long double s[4];     /* error scale components */
  int has;
} facc;

/* term = f(t) in S precision, as doubles */
static void map_float(forge_op op, const unsigned char* t, long double* v, long double* s) {
  switch (op) {
    case FORGE_OP_F32_SUM:
    case FORGE_OP_F32_LOGSUMEXP: {
      float x;
      memcpy(&x, t, 4);
      v[0] = x;
      s[0] = fabsl((long double)x);
      break;
    }
    case FORGE_OP_F32_SUMSQ: {
      float x;
      memcpy(&x, t, 4);
      float y = x * x;
      v[0] = y;
      s[0] = y;
      break;
    }
    case FORGE_OP_F64_SUM: {
      double x;
      memcpy(&x, t, 8);
      v[0] = x;
      s[0] = fabsl((long double)x);
      break;
    }
    case FORGE_OP_UF8_F32_SUM: {
      float x = orc_uf8_decode(*t);
      v[0] = x;
      s[0] = fabsl((long double)x);
      break;
    }
    case FORGE_OP_AFFINE_F32: {
      forge_affine_f32 a;
      memcpy(&a, t, 8);
      v[0] = a.a;
      v[1] = a.b;
      s[0] = fabsl((long double)a.a);
      s[1] = fabsl((long double)a.b);
      break;
    }
    case FORGE_OP_QUAT_F32: {
      forge_quat_f32 q;
      memcpy(&q, t, 16);
      v[0] = q.w;
      v[1] = q.x;
      v[2] = q.y;
      v[3] = q.z;
      long double nrm = sqrtl(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
      s[0] = s[1] = s[2] = s[3] = nrm;
      break;
    }
    default:
      break;
  }
}

/* acc = acc op term (acc is the older operand) */
static void fold_float(forge_op op, facc* acc, const long double* v, const long double* s) {
  if (!acc->has) {
    for (int k = 0; k < 4; ++k) {
      acc->v[k] = v[k];
      acc->s[k] = s[k];
    }
    acc->has = 1;
    return;
  }
  switch (op) {
    case FORGE_OP_F32_SUM:
    case FORGE_OP_F32_SUMSQ:
    case FORGE_OP_F64_SUM:
    case FORGE_OP_UF8_F32_SUM:
    case FORGE_OP_MV_F32_PLUS_TIMES:
    case FORGE_OP_MV_F64_PLUS_TIMES:
      acc->v[0] += v[0];
      acc->s[0] += s[0];
      break;
    case FORGE_OP_F32_LOGSUMEXP: { /* algebra.hpp:93-100, in extended precision */
      long double a = acc->v[0], b = v[0];
      if (isinf(a) && a < 0) {
        acc->v[0] = b;
      } else if (!(isinf(b) && b < 0)) {
        long double hi = a > b ? a : b, lo = a > b ? b : a;
        acc->v[0] = hi + log1pl(expl(lo - hi));
      }
      acc->s[0] = fabsl(acc->v[0]) + 1.0L;
      break;
    }
    case FORGE_OP_AFFINE_F32: { /* compose(p, q) = {q.a*p.a, q.a*p.b + q.b} */
      long double pa = acc->v[0], pb = acc->v[1];
      long double spa = acc->s[0], spb = acc->s[1];
      acc->v[0] = v[0] * pa;
      acc->v[1] = v[0] * pb + v[1];
      acc->s[0] = s[0] * spa;
      acc->s[1] = s[0] * spb + s[1];
      break;
    }
    case FORGE_OP_QUAT_F32: { /* algebra.hpp:37-44 with a = acc, b = term */
      long double aw = acc->v[0], ax = acc->v[1], ay = acc->v[2], az = acc->v[3];
      long double bw = v[0], bx = v[1], by = v[2], bz = v[3];
      acc->v[0] = aw * bw - ax * bx - ay * by - az * bz;
      acc->v[1] = aw * bx + ax * bw + ay * bz - az * by;
      acc->v[2] = aw * by - ax * bz + ay * bw + az * bx;
      acc->v[3] = aw * bz + ax * by - ay * bx + az * bw;
      for (int k = 0; k < 4; ++k) acc->s[k] = acc->s[k] * s[k];
      break;
    }
    default:
      break;
  }
}

static void facc_identity(forge_op op, facc* acc) {
  memset(acc, 0, sizeof *acc);
  acc->has = 1;
  switch (op) {
    case FORGE_OP_F32_LOGSUMEXP:
      acc->v[0] = -INFINITY;
      acc->s[0] = 1.0L;
      break;
    case FORGE_OP_AFFINE_F32:
      acc->v[0] = 1.0L;
      break;
    case FORGE_OP_QUAT_F32:
      acc->v[0] = 1.0L;
      break;
    default:
      break;
  }
}

/* S value carried as a float op accumulator start (carry-in). */
static void facc_from_s(forge_op op, const unsigned char* sraw, facc* acc) {
  long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
  if (op == FORGE_OP_UF8_F32_SUM) { /* S is f32 */
    float x;
    memcpy(&x, sraw, 4);
    v[0] = x;
    s[0] = fabsl((long double)x);
  } else if (op == FORGE_OP_F32_SUMSQ) {
    float x;
    memcpy(&x, sraw, 4);
    v[0] = x;
    s[0] = fabsl((long double)x);
  } else {
    map_float(op, sraw, v, s);
  }
  memset(acc, 0, sizeof *acc);
  fold_float(op, acc, v, s);
}

static void facc_to_s(forge_op op, const facc* acc, unsigned char* out, double* exact,
                      double* scale) {
  int nc = orc_float_components(op);
  for (int k = 0; k < nc; ++k) {
    if (exact) exact[k] = (double)acc->v[k];
    if (scale) scale[k] = (double)acc->s[k];
  }
  switch (op) {
    case FORGE_OP_F64_SUM:
    case FORGE_OP_MV_F64_PLUS_TIMES: {
      double d = (double)acc->v[0];
      memcpy(out, &d, 8);
      break;
    }
    case FORGE_OP_AFFINE_F32: {
      forge_affine_f32 a = {(float)acc->v[0], (float)acc->v[1]};
      memcpy(out, &a, 8);
      break;
    }
    case FORGE_OP_QUAT_F32: {
      forge_quat_f32 q = {(float)acc->v[0], (float)acc->v[1], (float)acc->v[2],
                          (float)acc->v[3]};
      memcpy(out, &q, 16);
      break;
    }
    default: {
      float f = (float)acc->v[0];
      memcpy(out, &f, 4);
      break;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* mapreduce (primitives.hpp:348-431)                                        */

int orc_mapreduce(forge_op op, const void* src, uint64_t n, uint64_t stride, void* out_S,
                  double* exact, double* scale) {
  const unsigned char* p = (const unsigned char*)src;
  uint32_t ts = t_size_of(op);
  if (stride == 0) stride = 1;
  if (orc_float_components(op)) {
    facc acc;
    if (n == 0) {
      facc_identity(op, &acc);
    } else {
      memset(&acc, 0, sizeof acc);
      for (uint64_t i = 0; i < n; ++i) {
        long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
        map_float(op, p + i * stride * ts, v, s);
        fold_float(op, &acc, v, s);
      }
    }
    facc_to_s(op, &acc, (unsigned char*)out_S, exact, scale);
    return 0;
  }
  sval acc = identity_of(op);
  for (uint64_t i = 0; i < n; ++i) {
    sval t = map_exact(op, p + i * stride * ts);
    acc = i == 0 ? t : combine_exact(op, acc, t);
  }
  memcpy(out_S, acc.raw, s_size_of(op));
  return 0;
}

/* Synthetic f32 inputs are integers times 2^-24 (gen_f32_sym / gen_f32_pos),
 * so their sums — and sums of |x| — are EXACT in int64 units of 2^-24 for any
 * n <= 2^38: the f32-sum oracle streams at integer speed (the long-double fold
 * costs ~60 ns per element; the 2^33-element BASELINE C5 size needs this). */
static int f32_sum_grid(forge_op op) { return op == FORGE_OP_F32_SUM; }
static int64_t f32_units(uint64_t u, int32_t variant) {
  const float v = variant == 1 ? gen_f32_pos(u) : gen_f32_sym(u);
  return (int64_t)llrintf(v * 16777216.0f); /* exact: |v| <= 1, 24-bit grid */
}

int orc_mapreduce_synthetic(forge_op op, uint64_t n, uint64_t seed, int32_t variant, void* out_S,
                            double* exact, double* scale) {
  unsigned char t[16];
  if (f32_sum_grid(op) && n > 0) {
    int64_t acc = 0, abs_acc = 0;
    /* integer sums are exact in any order: host threads may split the stream */
#pragma omp parallel for reduction(+ : acc, abs_acc) schedule(static)
    for (uint64_t i = 0; i < n; ++i) {
      const int64_t k = f32_units(orc_mix(seed ^ i), variant);
      acc += k;
      abs_acc += k < 0 ? -k : k;
    }
    const long double ex = (long double)acc / 16777216.0L;
    const float r = (float)ex;
    memcpy(out_S, &r, 4);
    if (exact) exact[0] = (double)ex;
    if (scale) scale[0] = (double)((long double)abs_acc / 16777216.0L);
    return 0;
  }
  if (orc_float_components(op)) {
    facc acc;
    if (n == 0) facc_identity(op, &acc);
    else memset(&acc, 0, sizeof acc);
    for (uint64_t i = 0; i < n; ++i) {
      gen_one(op, orc_mix(seed ^ i), i, variant, t);
      long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
      map_float(op, t, v, s);
      fold_float(op, &acc, v, s);
    }
    facc_to_s(op, &acc, (unsigned char*)out_S, exact, scale);
    return 0;
  }
  sval acc = identity_of(op);
  for (uint64_t i = 0; i < n; ++i) {
    gen_one(op, orc_mix(seed ^ i), i, variant, t);
    sval v = map_exact(op, t);
    acc = i == 0 ? v : combine_exact(op, acc, v);
  }
  memcpy(out_S, acc.raw, s_size_of(op));
  return 0;
}

/* ------------------------------------------------------------------------ */
/* scan (primitives.hpp:440-603)                                             */

int orc_scan(forge_op op, int32_t inclusive, const void* src, uint64_t n, const void* carry,
             void* dst_S, double* exact, double* scale) {
  const unsigned char* p = (const unsigned char*)src;
  unsigned char* d = (unsigned char*)dst_S;
  uint32_t ts = t_size_of(op), ss = s_size_of(op);
  int nc = orc_float_components(op);
  if (nc) {
    facc acc, ident;
    facc_identity(op, &ident);
    if (carry) facc_from_s(op, (const unsigned char*)carry, &acc);
    else memset(&acc, 0, sizeof acc);
    for (uint64_t i = 0; i < n; ++i) {
      long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
      map_float(op, p + i * ts, v, s);
      if (!inclusive) {
        const facc* cur = acc.has ? &acc : &ident; /* dst[0] = identity (:592) */
        facc_to_s(op, cur, d + i * ss, exact ? exact + i * nc : NULL,
                  scale ? scale + i * nc : NULL);
      }
      fold_float(op, &acc, v, s);
      if (inclusive)
        facc_to_s(op, &acc, d + i * ss, exact ? exact + i * nc : NULL,
                  scale ? scale + i * nc : NULL);
    }
    return 0;
  }
  sval acc;
  int has = 0;
  if (carry) {
    memset(&acc, 0, sizeof acc);
    memcpy(acc.raw, carry, ss);
    has = 1;
  }
  sval ident = identity_of(op);
  for (uint64_t i = 0; i < n; ++i) {
    sval t = map_exact(op, p + i * ts);
    if (!inclusive) memcpy(d + i * ss, (has ? acc : ident).raw, ss);
    acc = has ? combine_exact(op, acc, t) : t;
    has = 1;
    if (inclusive) memcpy(d + i * ss, acc.raw, ss);
  }
  return 0;
}

/* Streaming scan check.  idx == NULL: every output got_S[i], i < n.  Else the
 * outputs at the ascending positions idx[0..count) (got_S[k] is the output at
 * idx[k]); the stream stops after the last sampled position — how the
 * BASELINE C5 size (2^33 elements, 32 GiB of outputs) is checked without
 * copying the outputs to the host. */
static int64_t check_scan_stream(forge_op op, int32_t inclusive, uint64_t n, uint64_t seed, int32_t variant,
                                 const uint64_t* idx, uint64_t count, const void* got_S, double tol,
                                 double* max_err) {
  const unsigned char* g = (const unsigned char*)got_S;
  uint32_t ss = s_size_of(op);
  int nc = orc_float_components(op);
  unsigned char t[16];
  int64_t bad = 0;
  double worst = 0.0;
  uint64_t k = 0; /* next sample */
  const uint64_t end = idx ? (count ? idx[count - 1] + 1 : 0) : n;
  if (f32_sum_grid(op) && idx && count > 0) {
    /* Sampled check, exact integer prefix: chunk sums in parallel, exclusive
     * prefix over chunks, then every chunk checks its own samples. */
    enum { NCHUNK = 256 };
    static int64_t csum[NCHUNK + 1], cabs[NCHUNK + 1];
    const uint64_t per = (end + NCHUNK - 1) / NCHUNK;
#pragma omp parallel for schedule(dynamic)
    for (int c = 0; c < NCHUNK; ++c) {
      int64_t a = 0, b = 0;
      const uint64_t lo = (uint64_t)c * per, hi = lo + per < end ? lo + per : end;
      for (uint64_t i = lo; i < hi; ++i) {
        const int64_t kk = f32_units(orc_mix(seed ^ i), variant);
        a += kk;
        b += kk < 0 ? -kk : kk;
      }
      csum[c + 1] = a;
      cabs[c + 1] = b;
    }
    csum[0] = cabs[0] = 0;
    for (int c = 0; c < NCHUNK; ++c) {
      csum[c + 1] += csum[c];
      cabs[c + 1] += cabs[c];
    }
    int64_t nbad = 0;
    double w = 0.0;
#pragma omp parallel for schedule(dynamic) reduction(+ : nbad)
    for (int c = 0; c < NCHUNK; ++c) {
      const uint64_t lo = (uint64_t)c * per, hi = lo + per < end ? lo + per : end;
      uint64_t s0 = 0; /* first sample >= lo */
      { uint64_t L = 0, R = count; while (L < R) { uint64_t M = (L + R) / 2; if (idx[M] < lo) L = M + 1; else R = M; } s0 = L; }
      if (s0 >= count || idx[s0] >= hi) continue;
      int64_t a = csum[c], b = cabs[c];
      double lw = 0.0;
      uint64_t kk2 = s0;
      for (uint64_t i = lo; i < hi && kk2 < count; ++i) {
        const int64_t ex_a = a, ex_b = b;
        const int64_t u = f32_units(orc_mix(seed ^ i), variant);
        a += u;
        b += u < 0 ? -u : u;
        while (kk2 < count && idx[kk2] == i) {
          float gf;
          memcpy(&gf, g + kk2 * ss, 4);
          const int64_t ea = inclusive ? a : ex_a, eb = inclusive ? b : ex_b;
          const double ex = (double)((long double)ea / 16777216.0L);
          const double sc = (double)((long double)eb / 16777216.0L);
          const double err = fabs((double)gf - ex);
          const double rel = sc > 0 ? err / sc : (err > 0 ? INFINITY : 0.0);
          if (rel > lw || rel != rel) lw = rel != rel ? INFINITY : rel;
          if (!(err <= tol * sc)) ++nbad;
          ++kk2;
        }
      }
#pragma omp critical
      if (lw > w) w = lw;
    }
    bad = nbad;
    worst = w;
  } else if (f32_sum_grid(op)) {
    int64_t acc = 0, abs_acc = 0;
    int has = 0;
    for (uint64_t i = 0; i < end; ++i) {
      const int64_t kk = f32_units(orc_mix(seed ^ i), variant);
      const int64_t ex_acc = acc, ex_abs = abs_acc;
      const int ex_has = has;
      acc += kk;
      abs_acc += kk < 0 ? -kk : kk;
      has = 1;
      while (!idx || (k < count && idx[k] == i)) {
        float gf;
        memcpy(&gf, g + (idx ? k : i) * ss, 4);
        double ex, sc;
        if (inclusive) {
          ex = (double)((long double)acc / 16777216.0L);
          sc = (double)((long double)abs_acc / 16777216.0L);
        } else if (ex_has) {
          ex = (double)((long double)ex_acc / 16777216.0L);
          sc = (double)((long double)ex_abs / 16777216.0L);
        } else {
          ex = 0.0; /* identity */
          sc = 0.0;
        }
        const double err = fabs((double)gf - ex);
        const double rel = sc > 0 ? err / sc : (err > 0 ? INFINITY : 0.0);
        if (rel > worst || rel != rel) worst = rel != rel ? INFINITY : rel;
        if (!(err <= tol * sc)) ++bad;
        if (!idx) break;
        ++k;
      }
    }
  } else if (nc) {
    facc acc, ident;
    facc_identity(op, &ident);
    memset(&acc, 0, sizeof acc);
    for (uint64_t i = 0; i < end; ++i) {
      gen_one(op, orc_mix(seed ^ i), i, variant, t);
      long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
      map_float(op, t, v, s);
      if (inclusive) fold_float(op, &acc, v, s);
      while (!idx || (k < count && idx[k] == i)) {
        const unsigned char* gi = g + (idx ? k : i) * ss;
        const facc* cur = acc.has ? &acc : &ident;
        for (int c = 0; c < nc; ++c) {
          double got;
          if (op == FORGE_OP_F64_SUM) {
            memcpy(&got, gi, 8);
          } else {
            float gf;
            memcpy(&gf, gi + 4 * c, 4);
            got = gf;
          }
          double ex = (double)cur->v[c], sc = (double)cur->s[c];
          double err = fabs(got - ex);
          double rel = sc > 0 ? err / sc : (err > 0 ? INFINITY : 0.0);
          if (rel > worst || rel != rel) worst = rel != rel ? INFINITY : rel;
          if (!(err <= tol * sc)) {
            ++bad;
            break;
          }
        }
        if (!idx) break;
        ++k;
      }
      if (!inclusive) fold_float(op, &acc, v, s);
    }
  } else {
    sval acc = identity_of(op), ident = identity_of(op);
    int has = 0;
    for (uint64_t i = 0; i < end; ++i) {
      gen_one(op, orc_mix(seed ^ i), i, variant, t);
      sval v = map_exact(op, t);
      sval ex_before = has ? acc : ident;
      acc = has ? combine_exact(op, acc, v) : v;
      has = 1;
      while (!idx || (k < count && idx[k] == i)) {
        const unsigned char* gi = g + (idx ? k : i) * ss;
        if (memcmp(gi, inclusive ? acc.raw : ex_before.raw, ss) != 0) ++bad;
        if (!idx) break;
        ++k;
      }
    }
  }
  if (max_err) *max_err = worst;
  return bad;
}

int64_t orc_check_scan_synthetic(forge_op op, int32_t inclusive, uint64_t n, uint64_t seed,
                                 int32_t variant, const void* got_S, double tol,
                                 double* max_err) {
  return check_scan_stream(op, inclusive, n, seed, variant, NULL, 0, got_S, tol, max_err);
}

int64_t orc_check_scan_synthetic_at(forge_op op, int32_t inclusive, uint64_t seed, int32_t variant,
                                    const uint64_t* idx, uint64_t count, const void* got_at, double tol,
                                    double* max_err) {
  return check_scan_stream(op, inclusive, 0, seed, variant, idx, count, got_at, tol, max_err);
}

/* ------------------------------------------------------------------------ */
/* matvec / vecmat (primitives.hpp:775-807)                                  */

/* f(l, r) for the 2-D ops; the map result is an S value rounded as the
 * reference rounds it (f evaluated in S precision). */
static void map2(forge_op op, const unsigned char* l, const unsigned char* r, sval* exact_s,
                 long double* v, long double* s) {
  switch (op) {
    case FORGE_OP_MV_F32_PLUS_TIMES: {
      float a, b;
      memcpy(&a, l, 4);
      memcpy(&b, r, 4);
      float y = a * b;
      v[0] = y;
      s[0] = fabsl((long double)y);
      break;
    }
    case FORGE_OP_MV_F64_PLUS_TIMES: {
      double a, b;
      memcpy(&a, l, 8);
      memcpy(&b, r, 8);
      double y = a * b;
      v[0] = y;
      s[0] = fabsl((long double)y);
      break;
    }
    case FORGE_OP_MV_F32_MIN_PLUS:
    case FORGE_OP_MV_F32_MAX_PLUS: {
      float a, b;
      memcpy(&a, l, 4);
      memcpy(&b, r, 4);
      memset(exact_s, 0, sizeof *exact_s);
      exact_s->f = a + b;
      break;
    }
    case FORGE_OP_MV_I32_PLUS_TIMES: {
      uint32_t a, b;
      memcpy(&a, l, 4);
      memcpy(&b, r, 4);
      memset(exact_s, 0, sizeof *exact_s);
      exact_s->u = a * b;
      break;
    }
    case FORGE_OP_MV_MAT2_U32: {
      forge_mat2_u32 a, b;
      memcpy(&a, l, 16);
      memcpy(&b, r, 16);
      memset(exact_s, 0, sizeof *exact_s);
      exact_s->m2 = mat2_mul(a, b);
      break;
    }
    default:
      break;
  }
}

static int is_binary(forge_op op) { return op >= FORGE_OP_MV_F32_PLUS_TIMES && op < FORGE_OP_MV_END_; }

/* One output: fold over k of f(left(k), right(k)) where for matvec
 * left = x[i], right = A[i,j]; for vecmat left = A[i,j], right = x[j]. */
static void mat_fold(forge_op op, const unsigned char* A, uint64_t a_first, uint64_t a_step,
                     const unsigned char* x, int x_left, uint64_t len, unsigned char* out,
                     double* exact, double* scale) {
  uint32_t ts = t_size_of(op), ss = s_size_of(op);
  int nc = orc_float_components(op);
  if (!is_binary(op)) { /* mapreduce_2d: unary map on A elements */
    if (nc) {
      facc acc;
      if (len == 0) facc_identity(op, &acc);
      else memset(&acc, 0, sizeof acc);
      for (uint64_t k = 0; k < len; ++k) {
        long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
        map_float(op, A + (a_first + k * a_step) * ts, v, s);
        fold_float(op, &acc, v, s);
      }
      facc_to_s(op, &acc, out, exact, scale);
    } else {
      sval acc = identity_of(op);
      for (uint64_t k = 0; k < len; ++k) {
        sval t = map_exact(op, A + (a_first + k * a_step) * ts);
        acc = k == 0 ? t : combine_exact(op, acc, t);
      }
      memcpy(out, acc.raw, ss);
    }
    return;
  }
  if (nc) {
    facc acc;
    if (len == 0) facc_identity(op, &acc);
    else memset(&acc, 0, sizeof acc);
    for (uint64_t k = 0; k < len; ++k) {
      const unsigned char* a = A + (a_first + k * a_step) * ts;
      const unsigned char* xv = x + k * ts;
      long double v[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
      sval dummy;
      map2(op, x_left ? xv : a, x_left ? a : xv, &dummy, v, s);
      fold_float(op, &acc, v, s);
    }
    facc_to_s(op, &acc, out, exact, scale);
  } else {
    sval acc = identity_of(op);
    for (uint64_t k = 0; k < len; ++k) {
      const unsigned char* a = A + (a_first + k * a_step) * ts;
      const unsigned char* xv = x + k * ts;
      long double v[4], s[4];
      sval t;
      map2(op, x_left ? xv : a, x_left ? a : xv, &t, v, s);
      acc = k == 0 ? t : combine_exact(op, acc, t);
    }
    memcpy(out, acc.raw, ss);
  }
}

int orc_matvec(forge_op op, const void* A, uint64_t n, uint64_t p, const void* x, void* y_S,
               double* exact, double* scale) {
  uint32_t ss = s_size_of(op);
  int nc = orc_float_components(op);
  for (uint64_t j = 0; j < p; ++j)
    mat_fold(op, (const unsigned char*)A, j * n, 1, (const unsigned char*)x, 1, n,
             (unsigned char*)y_S + j * ss, exact ? exact + j * nc : NULL,
             scale ? scale + j * nc : NULL);
  return 0;
}

int orc_vecmat(forge_op op, const void* A, uint64_t n, uint64_t p, const void* x, void* z_S,
               double* exact, double* scale) {
  uint32_t ss = s_size_of(op);
  int nc = orc_float_components(op);
  for (uint64_t i = 0; i < n; ++i)
    mat_fold(op, (const unsigned char*)A, i, n, (const unsigned char*)x, 0, p,
             (unsigned char*)z_S + i * ss, exact ? exact + i * nc : NULL,
             scale ? scale + i * nc : NULL);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* vload_pattern (intrinsics.hpp:198-211): greedy power-of-two segments, each
 * aligned to its own size at the running element offset.                  */

int orc_vload_pattern(uint64_t offset, uint32_t nitem, uint32_t* segs, uint32_t* count) {
  if (nitem != 1 && nitem != 2 && nitem != 4 && nitem != 8 && nitem != 16)
    return FORGE_ERR_INVALID_NITEM;
  uint64_t o = offset;
  uint32_t rem = nitem, c = 0;
  while (rem > 0) {
    uint32_t by_align = nitem;
    if (o != 0) {
      uint64_t low = o & (~o + 1); /* 2^ctz(o) */
      by_align = low < nitem ? (uint32_t)low : nitem;
    }
    uint32_t by_rem = 1;
    while (by_rem * 2 <= rem) by_rem *= 2;
    uint32_t s = by_align < by_rem ? by_align : by_rem;
    segs[c++] = s;
    o += s;
    rem -= s;
  }
  *count = c;
  return 0;
}
