/*
 * oracle.h — CPU restatement of the reference primitive semantics.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (libforge.so, the
 * paper_2603_18695_b200 package) may link, load or call this code; it is the
 * checker used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg.  Every function cites the /root/reference/proj file:line it restates.
 *
 * Parity pinning: the restatement is checked (tests/test_oracle.py) against
 *   - the SPEC.md known-answer vectors (SPEC.md:220-222, 304-306, 314-315,
 *     324-325, 334-335, 342, 361-362, 422-435), and
 *   - the reference VM itself, compiled from /root/reference by oracle/ref/
 *     into oracle/_ref/libforge_ref.so (bit-exact for exact operators, within
 *     the stated tolerance for floating point); committed golden fixtures in
 *     tests/golden/ carry those reference outputs to machines without
 *     /root/reference.
 */
#ifndef FORGE_ORACLE_H_
#define FORGE_ORACLE_H_

#include <stdint.h>

#include "../include/forge.h"

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64 finaliser (the same mixing as proj/src/prng.hpp:12-17). */
uint64_t orc_mix(uint64_t x);

/* Synthetic input generator; bit-identical to the device
 * generator forge_dev_fill_synthetic.  Fills n elements of the op's T. */
int orc_fill_synthetic(forge_op op, void* dst, uint64_t n, uint64_t seed, uint64_t index_base,
                       int32_t variant);

/* Number of scalar components compared for floating-point outputs of op
 * (0 for exact operators, whose S outputs are compared bit for bit). */
int orc_float_components(forge_op op);

/* mapreduce (primitives.hpp:348-431): sequential fold of f(src[i*stride]).
 * out_S receives the S result (for float ops: the f64-accumulated value
 * rounded to S); exact/scale (nullable, orc_float_components doubles each)
 * receive the 64-bit-accumulated value and the error scale sum |terms|.
 * Returns 0, or FORGE_ERR_MISSING_IDENTITY for empty input without identity
 * semantics handled by the caller. */
int orc_mapreduce(forge_op op, const void* src, uint64_t n, uint64_t stride, void* out_S,
                  double* exact, double* scale);

/* scan (primitives.hpp:440-603): inclusive dst[i] = fold f(src[0..i]);
 * exclusive dst[0] = identity (or carry), dst[i] = fold f(src[0..i-1])
 * (primitives.hpp:587-595).  carry (nullable, S) is folded in front. */
int orc_scan(forge_op op, int32_t inclusive, const void* src, uint64_t n, const void* carry,
             void* dst_S, double* exact, double* scale);

/* matvec (primitives.hpp:776-791) y[j] = op_i f(x[i], A[i,j]) and vecmat
 * (primitives.hpp:795-807) z[i] = op_j f(A[i,j], x[j]); A column-major n x p.
 * x == NULL means uses_vector = false with a 1-D op applied to A elements
 * (mapreduce_2d, primitives.hpp:814-836). */
int orc_matvec(forge_op op, const void* A, uint64_t n, uint64_t p, const void* x, void* y_S,
               double* exact, double* scale);
int orc_vecmat(forge_op op, const void* A, uint64_t n, uint64_t p, const void* x, void* z_S,
               double* exact, double* scale);

/* vload_pattern (intrinsics.hpp:198-211, intrinsics.cpp:29-33). */
int orc_vload_pattern(uint64_t offset, uint32_t nitem, uint32_t* segs, uint32_t* count);

/* Streaming full-size checks without materialising the input (inputs from the
 * synthetic generator): mapreduce over n generated elements. */
int orc_mapreduce_synthetic(forge_op op, uint64_t n, uint64_t seed, int32_t variant, void* out_S,
                            double* exact, double* scale);

/* Compares a device scan output against the sequential oracle over generated
 * input, streaming.  Returns the number of mismatching elements (exact ops:
 * bitwise; float ops: |got-exact| > tol*scale); *max_err receives the largest
 * err/scale seen. */
int64_t orc_check_scan_synthetic(forge_op op, int32_t inclusive, uint64_t n, uint64_t seed,
                                 int32_t variant, const void* got_S, double tol, double* max_err);
/* Same check at ascending sampled positions idx[0..count): got_at[k] is the
 * output at idx[k] (streams up to the last position). */
int64_t orc_check_scan_synthetic_at(forge_op op, int32_t inclusive, uint64_t seed, int32_t variant,
                                    const uint64_t* idx, uint64_t count, const void* got_at, double tol,
                                    double* max_err);

/* UnitFloat8 (algebra.hpp:15-28). */
float orc_uf8_decode(uint8_t code);
uint8_t orc_uf8_encode(float x);

#ifdef __cplusplus
}
#endif

#endif
