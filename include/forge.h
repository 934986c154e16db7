/*
 * forge.h — the C-ABI drop-in boundary of the B200 primitive layer.
 *
 * The reference declares this surface but never ships it: proj/src/CMakeLists.txt:13-17
 * builds `libforge.so` from `capi.cpp`, "the extern-C surface declared in
 * include/forge/forge.h"; neither file exists in /root/reference.  This header is
 * that surface, re-designed for sm_100a: every entry point below names the
 * reference C++ interface it replaces (file:line under /root/reference/proj).
 *
 * Two layers:
 *   1. Machine-level calls (forge_machine_*, forge_scan, forge_mapreduce, ...)
 *      mirror forge::Machine / forge::prim with BufferIds, Views, Workspaces and
 *      LaunchReports.  Launches are synchronous, like Machine::launch
 *      (machine.hpp:175-178).
 *   2. Device-pointer calls (forge_dev_*) take raw device pointers plus a
 *      cudaStream_t (as void*) and are stream-ordered and asynchronous; the
 *      sharded multi-GPU layer and torch-tensor callers use these.
 *
 * Arbitrary (T, S, f, op) are served by the header templates in
 * include/forge/primitives.hpp (instantiated in the caller's nvcc TU); across
 * the C-ABI only the fixed operator menu `forge_op` below is available.  Both
 * go through the same kernel source (the headers under include/forge/cuda/).
 *
 * Status codes: 0 = ok; 1 + forge::ErrorCode for host-side validation errors
 * (error.hpp:10-19, same order); FORGE_ERR_DEVICE_FAULT when the device launch
 * failed (the reference reports device faults through LaunchReport.ok=false,
 * error.hpp:8-9; the report, when passed, is filled as well).  The message of the
 * last failure on the calling thread is returned by forge_last_error().
 */
#ifndef FORGE_H_
#define FORGE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FORGE_ABI_VERSION 1

typedef enum forge_status {
  FORGE_OK = 0,
  FORGE_ERR_INVALID_ARGUMENT = 1,    /* ErrorCode::InvalidArgument   error.hpp:11 */
  FORGE_ERR_INVALID_DESCRIPTOR = 2,  /* ErrorCode::InvalidDescriptor error.hpp:12 */
  FORGE_ERR_INVALID_NITEM = 3,       /* ErrorCode::InvalidNitem      error.hpp:13 */
  FORGE_ERR_MISSING_IDENTITY = 4,    /* ErrorCode::MissingIdentity   error.hpp:14 */
  FORGE_ERR_WORKSPACE_TOO_SMALL = 5, /* ErrorCode::WorkspaceTooSmall error.hpp:15 */
  FORGE_ERR_DIMENSION_MISMATCH = 6,  /* ErrorCode::DimensionMismatch error.hpp:16 */
  FORGE_ERR_PARSE_ERROR = 7,         /* ErrorCode::ParseError        error.hpp:17 */
  FORGE_ERR_UNSUPPORTED = 8,         /* ErrorCode::Unsupported       error.hpp:18 */
  FORGE_ERR_DEVICE_FAULT = 100,      /* LaunchReport{ok=false}       machine.hpp:82-90 */
  FORGE_ERR_NO_DEVICE = 101          /* no CUDA device / driver: the library never falls back to the CPU */
} forge_status;

/* ---------------------------------------------------------------------------
 * The operator menu.  A forge_op fixes (T, S, f, op, identity, commutative) the
 * way a SemiringSpec does (primitives.hpp:92-104).  Element types:
 *   forge_affine_f32  {float a, b}      x -> a*x + b; compose(p, q) = q after p
 *   forge_argmax      {float v; int32 i} max v, ties to the smaller i
 *   forge_mat2_u32    {uint32 m[4]}      algebra.hpp:52-65 (row-major, wrapping)
 *   forge_quat_f32    {float w,x,y,z}    algebra.hpp:33-46 (Hamilton product)
 *   UnitFloat8        uint8 code         algebra.hpp:15-28, decode = -1 + 2c/255
 */
typedef enum forge_op {
  /* 1-D semirings (scan, mapreduce, mapreduce_2d): f: T -> S */
  FORGE_OP_F32_SUM = 0,         /* T=S=f32  f=id   op=+    id=0      commutative */
  FORGE_OP_F32_SUMSQ = 1,       /* T=S=f32  f=x*x  op=+    id=0      commutative */
  FORGE_OP_F32_MAX = 2,         /* T=S=f32  f=id   op=max  id=-inf   commutative */
  FORGE_OP_F32_MIN = 3,         /* T=S=f32  f=id   op=min  id=+inf   commutative */
  FORGE_OP_F64_SUM = 4,         /* T=S=f64  f=id   op=+    id=0      commutative */
  FORGE_OP_I32_SUM = 5,         /* T=S=i32  f=id   op=+ (wrapping)   commutative */
  FORGE_OP_I32_MAX = 6,         /* T=S=i32  f=id   op=max  id=INT32_MIN          */
  FORGE_OP_I32_MIN = 7,         /* T=S=i32  f=id   op=min  id=INT32_MAX          */
  FORGE_OP_U32_SUM = 8,         /* T=S=u32  f=id   op=+ (wrapping)               */
  FORGE_OP_I64_SUM = 9,         /* T=S=i64  f=id   op=+ (wrapping)               */
  FORGE_OP_AFFINE_F32 = 10,     /* T=S=affine  op=compose  id={1,0}  NOT commutative */
  FORGE_OP_ARGMAX_F32I32 = 11,  /* T=S=argmax  op=argmax   id={-inf,INT32_MAX} commutative */
  FORGE_OP_MAT2_U32 = 12,       /* T=S=mat2    op=mat2_mul id=I      NOT commutative */
  FORGE_OP_QUAT_F32 = 13,       /* T=S=quat    op=qmul     id=1      NOT commutative */
  FORGE_OP_UF8_F32_SUM = 14,    /* T=u8 (UnitFloat8) S=f32 f=decode op=+ commutative */
  FORGE_OP_F32_LOGSUMEXP = 15,  /* T=S=f32  op=log_sum_exp (algebra.hpp:93-100) id=-inf */
  FORGE_OP_1D_COUNT_ = 16,

  /* 2-D semirings (matvec, vecmat): f: T x T -> S.  matvec calls f(x[i], A[i,j]),
   * vecmat calls f(A[i,j], x[j]) (primitives.hpp:775-807). */
  FORGE_OP_MV_F32_PLUS_TIMES = 32, /* f=a*b  op=+    id=0     commutative (gemv/gevm) */
  FORGE_OP_MV_F32_MIN_PLUS = 33,   /* f=a+b  op=min  id=+inf  commutative (tropical)  */
  FORGE_OP_MV_F32_MAX_PLUS = 34,   /* f=a+b  op=max  id=-inf  commutative             */
  FORGE_OP_MV_I32_PLUS_TIMES = 35, /* f=a*b  op=+ wrapping    commutative (exact)     */
  FORGE_OP_MV_F64_PLUS_TIMES = 36, /* f=a*b  op=+    id=0     commutative             */
  FORGE_OP_MV_MAT2_U32 = 37,       /* f=mat2_mul(a,b) op=mat2_mul  NOT commutative (ordered path) */
  FORGE_OP_MV_END_ = 38
} forge_op;

typedef struct forge_affine_f32 { float a, b; } forge_affine_f32;
typedef struct forge_argmax { float v; int32_t i; } forge_argmax;
typedef struct forge_mat2_u32 { uint32_t m[4]; } forge_mat2_u32;
typedef struct forge_quat_f32 { float w, x, y, z; } forge_quat_f32;

/* Static facts about an op: element sizes, identity availability, commutativity,
 * and whether it is a 1-D (unary map) or 2-D (binary map) semiring. */
typedef struct forge_op_info {
  uint32_t t_size;      /* sizeof(T) */
  uint32_t s_size;      /* sizeof(S) */
  uint32_t commutative; /* SemiringSpec::commutative (primitives.hpp:97) */
  uint32_t binary;      /* 1: f takes (T, T) (matvec/vecmat), 0: f takes T */
  const char* name;
} forge_op_info;
int forge_get_op_info(forge_op op, forge_op_info* out);

/* The semiring as a value: the op plus whether its identity is supplied.  An
 * op without identity behaves like SemiringSpec{identity = nullopt}: exclusive
 * scan and empty reductions raise MissingIdentity (primitives.hpp:359, 446, 742). */
typedef struct forge_semiring {
  forge_op op;
  int32_t has_identity;
} forge_semiring;

/* ---------------------------------------------------------------------------
 * Host-side types mirrored from the reference. */

/* ArchParams (primitives.hpp:16-60).  warp_width must be 32 on B200 (64 raises
 * Unsupported); geometry fields are validated like the reference and otherwise
 * advisory: the sm_100a kernels pick their own tiles. */
typedef struct forge_arch_params {
  uint32_t warp_width;
  uint32_t mapreduce_blocks;
  uint32_t threads_per_block;
  uint32_t nitem_scan;
  uint32_t nitem_copy;
  uint32_t lookback_window;
  uint32_t matvec_wide_warp_cols;
  uint32_t matvec_wide_block_threads;
  uint64_t matvec_wide_min_outputs;
} forge_arch_params;
void forge_arch_params_default(forge_arch_params* out);

typedef int32_t forge_buffer_id; /* BufferId (machine.hpp:130) */

/* View<T> (intrinsics.hpp:19-35): offset/length/stride in elements of buf. */
typedef struct forge_view {
  forge_buffer_id buf;
  uint64_t offset;
  uint64_t length;
  uint64_t stride;
} forge_view;

/* Workspace (primitives.hpp:180-195). */
typedef struct forge_workspace {
  forge_buffer_id tile_aggregate, tile_prefix, tile_flag, partials, flags, result;
  uint64_t tiles, slots;
} forge_workspace;

/* FaultKind (machine.hpp:50-60), same order. */
typedef enum forge_fault_kind {
  FORGE_FAULT_NONE = 0,
  FORGE_FAULT_OUT_OF_BOUNDS,
  FORGE_FAULT_STEP_BUDGET_EXCEEDED,
  FORGE_FAULT_BARRIER_DIVERGENCE,
  FORGE_FAULT_MISALIGNED_VECTOR_ACCESS,
  FORGE_FAULT_SHARED_MEMORY_EXHAUSTED,
  FORGE_FAULT_LANE_OUT_OF_RANGE,
  FORGE_FAULT_NON_UNIFORM_WARP_CALL,
  FORGE_FAULT_INTERNAL
} forge_fault_kind;

/* LaunchReport (machine.hpp:82-90).  wall_seconds is the CUDA-event time of the
 * primitive's device work (kernel launches only, not the host readback). */
typedef struct forge_launch_report {
  int32_t ok;
  int32_t fault_kind;
  uint64_t steps;       /* kernels launched by the primitive */
  double wall_seconds;
  char detail[240];
} forge_launch_report;

/* Primitive (primitives.hpp:176), for forge_required_workspace. */
typedef enum forge_primitive {
  FORGE_PRIM_SCAN = 0,
  FORGE_PRIM_MAPREDUCE = 1,
  FORGE_PRIM_MATVEC = 2,
  FORGE_PRIM_VECMAT = 3,
  FORGE_PRIM_VCOPY = 4,
  FORGE_PRIM_MAPREDUCE_2D = 5
} forge_primitive;

/* ReduceAxis (primitives.hpp:809). */
typedef enum forge_reduce_axis { FORGE_AXIS_ROWS = 0, FORGE_AXIS_COLS = 1 } forge_reduce_axis;

const char* forge_last_error(void);
int forge_abi_version(void);
int forge_device_count(int* out);

/* ---------------------------------------------------------------------------
 * Machine (machine.hpp:142-184): one CUDA device + one stream + a buffer table.
 * Buffers are zero-initialised device allocations (machine.cpp:968-986) with a
 * base alignment (default max(4096, bit_ceil(elem size)), machine.cpp:20,972). */
typedef struct forge_machine forge_machine;

int forge_machine_create(int device, forge_machine** out);                    /* Machine::Machine */
int forge_machine_destroy(forge_machine* m);                                  /* Machine::~Machine */
int forge_machine_stream(forge_machine* m, void** cuda_stream);
int forge_machine_synchronize(forge_machine* m);

/* Machine::create_buffer (machine.hpp:153-154) with the element given as a
 * descriptor literal (bitstype.hpp:58-63): "f32", "tuple(f32,u32)",
 * "struct(u8@0,f64@8,u16@16; size=24)". */
int forge_create_buffer(forge_machine* m, const char* descriptor, uint64_t length,
                        uint32_t base_alignment, forge_buffer_id* out);
int forge_destroy_buffer(forge_machine* m, forge_buffer_id id);               /* machine.hpp:155 */
int forge_buffer_length(forge_machine* m, forge_buffer_id id, uint64_t* out); /* machine.hpp:157 */
int forge_buffer_elem_size(forge_machine* m, forge_buffer_id id, uint32_t* out);
int forge_buffer_alignment(forge_machine* m, forge_buffer_id id, uint32_t* out);
int forge_buffer_device_ptr(forge_machine* m, forge_buffer_id id, void** out);
/* write_bytes/read_bytes/fill_zero (machine.hpp:162-164): synchronous host copies.
 * Pinned host memory gives full PCIe bandwidth; pageable memory works too. */
int forge_write_bytes(forge_machine* m, forge_buffer_id id, uint64_t elem_offset,
                      const void* src, uint64_t bytes);
int forge_read_bytes(forge_machine* m, forge_buffer_id id, uint64_t elem_offset, void* dst,
                     uint64_t bytes);
int forge_fill_zero(forge_machine* m, forge_buffer_id id);

/* Descriptor literals (bitstype.hpp:58-67). */
int forge_descriptor_info(const char* descriptor, uint32_t* size, uint32_t* alignment,
                          char* canonical, uint64_t canonical_cap);
/* value_bytes_equal (bitstype.hpp:70-71): equality on non-padding bytes. */
int forge_value_bytes_equal(const char* descriptor, const void* a, const void* b, int32_t* equal);

/* ---------------------------------------------------------------------------
 * Workspaces (primitives.hpp:246-300). */
int forge_required_workspace(forge_primitive prim, uint32_t accum_size, uint64_t n,
                             uint64_t p_cols, const forge_arch_params* params, uint64_t* bytes);
int forge_make_scan_workspace(forge_machine* m, forge_op op, uint64_t n,
                              const forge_arch_params* params, forge_workspace* out);
int forge_make_mapreduce_workspace(forge_machine* m, forge_op op,
                                   const forge_arch_params* params, forge_workspace* out);
int forge_make_mat_workspace(forge_machine* m, forge_op op, uint64_t reduce_len, uint64_t outputs,
                             const forge_arch_params* params, forge_workspace* out);
int forge_workspace_release(forge_machine* m, forge_workspace* ws);          /* Workspace::release */

/* ---------------------------------------------------------------------------
 * Primitives (primitives.hpp).  `report` may be NULL. */

/* scan (primitives.hpp:440-443): inclusive dst[i] = f(src[0]) op ... op f(src[i]);
 * exclusive dst[0] = identity, dst[i] = fold of f(src[0..i-1]). */
int forge_scan(forge_machine* m, forge_semiring spec, forge_view src, forge_view dst,
               int32_t inclusive, forge_workspace* ws, const forge_arch_params* params,
               forge_launch_report* report);

/* mapreduce (primitives.hpp:348-351): *out_host = fold of f(src[i]); the op must
 * be commutative (primitives.hpp:353-355). */
int forge_mapreduce(forge_machine* m, forge_semiring spec, forge_view src, forge_workspace* ws,
                    const forge_arch_params* params, void* out_host,
                    forge_launch_report* report);

/* matvec (primitives.hpp:776-791): y[j] = op_i f(x[i], A[i,j]); A n x p column-major. */
int forge_matvec(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n,
                 uint64_t p_cols, forge_view x, forge_view y, forge_workspace* ws,
                 const forge_arch_params* params, forge_launch_report* report,
                 int32_t uses_vector);

/* vecmat (primitives.hpp:795-807): z[i] = op_j f(A[i,j], x[j]). */
int forge_vecmat(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n,
                 uint64_t p_cols, forge_view x, forge_view z, forge_workspace* ws,
                 const forge_arch_params* params, forge_launch_report* report,
                 int32_t uses_vector);

/* mapreduce_2d (primitives.hpp:814-836): Rows -> one value per column, Cols ->
 * one value per row; spec is a 1-D op. */
int forge_mapreduce_2d(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n,
                       uint64_t p_cols, forge_reduce_axis axis, forge_view out,
                       forge_workspace* ws, const forge_arch_params* params,
                       forge_launch_report* report);

/* vcopy (primitives.hpp:305-341): dst = src bit-exactly; element type from the buffer. */
int forge_vcopy(forge_machine* m, forge_view src, forge_view dst, uint32_t nitem,
                const forge_arch_params* params, forge_launch_report* report);

/* MutationFlags (primitives.hpp:64-67), the reference's ordering ablation, for
 * the calling thread's subsequent forge_scan / forge_dev_scan calls.  TEST ONLY:
 * relax_scan_flag = 1 makes the scan accept tile states left by EARLIER launches
 * on the same workspace (the epoch tag is ignored), a deliberately broken
 * publication protocol that the relaunch stress tests must detect
 * (tests/test_gpu_stress.py).  relax_mapreduce_flag is accepted and ignored: the
 * B200 mapreduce never waits on another block's flag.  (0, 0) restores the
 * product protocol. */
int forge_set_mutation_flags(int32_t relax_scan_flag, int32_t relax_mapreduce_flag);

/* Adversarial schedule for the calling thread's subsequent scans, the B200
 * counterpart of the reference simulator's seeded schedules (ScheduleSeed,
 * machine.hpp:122-128).  TEST ONLY: seed != 0 makes a pseudo-random 1/8 of the
 * tiles (chosen by the seed) wait delay_ns before publishing their aggregate,
 * so their successors poll unpublished states.  Results are unchanged (the
 * protocol waits); without it B200 CTAs publish in ticket order and the
 * ablation above is never exercised.  seed = 0 turns it off. */
int forge_set_schedule_perturbation(uint64_t seed, uint32_t delay_ns);

/* vload_pattern (intrinsics.hpp:190, intrinsics.cpp:29-33). segs has room for 16. */
int forge_vload_pattern(uint64_t offset, uint32_t nitem, uint32_t* segs, uint32_t* count);

/* Ordering litmus tests (forge::lit, include/forge/litmus.hpp; reference
 * proj/include/forge/litmus.hpp, proj/src/litmus.cpp:169-350).  The text format
 * of parse_litmus ("blocks=<n> cells=<k>", "B<i>: st|ld <cell> [rel|acq|rlx]
 * [=<imm>]", "assert <expr>").  forge_litmus_parse only validates (no device
 * needed; FORGE_ERR_PARSE_ERROR with the message in forge_last_error()).
 * forge_litmus_run executes instances seed_begin .. seed_end-1 on the GPU (each
 * block of the program a CTA on its own SM) and fills `out`; `histogram` (may
 * be NULL) receives "<count>\t<outcome>\n" lines, most frequent first, cut
 * at histogram_cap bytes (always NUL-terminated when histogram_cap > 0). */
typedef struct forge_litmus_result {
  uint64_t seeds_run, assert_violations, faults, distinct_outcomes;
} forge_litmus_result;
int forge_litmus_parse(const char* spec_text);
int forge_litmus_run(const char* spec_text, uint64_t seed_begin, uint64_t seed_end, forge_litmus_result* out,
                     char* histogram, uint64_t histogram_cap);

/* ---------------------------------------------------------------------------
 * Device-pointer layer: stream-ordered, asynchronous, no host synchronisation.
 * `stream` is a cudaStream_t (NULL = the legacy default stream).  `ws` is caller
 * device memory of at least forge_dev_workspace_bytes(...) bytes (full speed;
 * a scan also accepts less, down to packed tile states), zeroed once before
 * first use (cudaMemset); the kernels leave it re-usable.  One workspace may
 * serve several primitives and shapes in turn: the library re-zeroes the part
 * a layout needs when the workspace last served another layout.  A workspace
 * must not be shared by launches in flight at the same time. */
int forge_dev_workspace_bytes(forge_primitive prim, forge_op op, uint64_t n, uint64_t p_cols,
                              uint64_t* bytes);

/* One-kernel mapreduce; the S result is written to out_dev (device memory). */
int forge_dev_mapreduce(forge_op op, const void* src, uint64_t n, void* out_dev, void* ws,
                        uint64_t ws_bytes, void* stream);

/* Order-preserving reduction over a contiguous range for any associative op
 * (commutativity not required); used for shard totals of the sharded scan. */
int forge_dev_reduce_ordered(forge_op op, const void* src, uint64_t n, void* out_dev, void* ws,
                             uint64_t ws_bytes, void* stream);

/* Single-pass decoupled look-back scan.  carry_in_dev (nullable) is an S value
 * folded in front of every prefix (the exclusive prefix of earlier shards);
 * total_out_dev (nullable) receives the inclusive total of the whole range
 * (carry included). */
int forge_dev_scan(forge_op op, int32_t inclusive, const void* src, void* dst, uint64_t n,
                   const void* carry_in_dev, void* total_out_dev, void* ws, uint64_t ws_bytes,
                   void* stream);

/* gevm / gemv over column-major A (n x p). */
int forge_dev_matvec(forge_op op, const void* A, uint64_t n, uint64_t p_cols, const void* x,
                     void* y, void* ws, uint64_t ws_bytes, void* stream);
int forge_dev_vecmat(forge_op op, const void* A, uint64_t n, uint64_t p_cols, const void* x,
                     void* z, void* ws, uint64_t ws_bytes, void* stream);
/* The same over an n x p block of a larger column-major matrix whose columns
 * are `lda` >= n elements apart (0 = n): A points at the block's first element.
 * A row block [lo, hi) of a global n_g x p matrix G is (G + lo, hi - lo, p,
 * lda = n_g) — the vecmat shard of SURVEY.md §8(e), consumed in place. */
int forge_dev_matvec_lda(forge_op op, const void* A, uint64_t n, uint64_t p_cols, uint64_t lda,
                         const void* x, void* y, void* ws, uint64_t ws_bytes, void* stream);
int forge_dev_vecmat_lda(forge_op op, const void* A, uint64_t n, uint64_t p_cols, uint64_t lda,
                         const void* x, void* z, void* ws, uint64_t ws_bytes, void* stream);

/* Fold of values[0..count-1] in index order (the rank-order fold of the sharded
 * exchange).  exclusive_upto >= 0 folds only values[0..exclusive_upto-1] and
 * writes *has_out_dev = 0 when that range is empty. */
int forge_dev_fold(forge_op op, const void* values_dev, uint32_t count, int32_t exclusive_upto,
                   void* out_dev, int32_t* has_out_dev, void* stream);

/* Bandwidth calibration copy (vcopy's device kernel) of `bytes` bytes. */
int forge_dev_copy(const void* src, void* dst, uint64_t bytes, void* stream);

/* Deterministic synthetic input, bit-identical to
 * oracle/oracle.c's generator: element i of the op's T is a function of
 * splitmix64(seed ^ (index_base + i)). */
int forge_dev_fill_synthetic(forge_op op, void* dst, uint64_t n, uint64_t seed,
                             uint64_t index_base, int32_t variant, void* stream);

/* ---------------------------------------------------------------------------
 * Single-process multi-GPU sharding for C / C++ callers.
 * The reference has no multi-device layer (one Machine = one simulated device,
 * machine.hpp:139-141); these calls shard the primitives across the GPUs of
 * one node, one shard per device, shards in rank order.
 *
 * forge_group_create(devices, count): count ordinals, rank r on devices[r].
 *   All distinct -> an NCCL clique (ncclCommInitAll over NVLink / NVSwitch;
 *   libnccl.so.2 is opened at first use, FORGE_ERR_UNSUPPORTED without it).
 *   All the same -> an EMULATED group: G shards on one GPU running the same
 *   exchange logic, the all-gather done by device copies (1-GPU test boxes).
 *   Anything else -> InvalidArgument.  The group owns one stream per shard;
 *   the sharded calls are stream-ordered on those streams (no host sync,
 *   except forge_sharded_mapreduce's host result) — forge_group_synchronize
 *   waits for them.  One group serves one sharded call at a time.
 *
 * Arrays are indexed by rank: src[r] / dst[r] / ws[r] are device pointers on
 * shard r's device, ws_bytes[r] >= forge_dev_workspace_bytes for that shard.
 * Shard r of a length-`total` array is forge_shard_range(total, r, G). */
typedef struct forge_group forge_group;

int forge_shard_range(uint64_t total, int32_t rank, int32_t count, uint64_t* lo, uint64_t* hi);
int forge_group_create(const int32_t* devices, int32_t count, forge_group** out);
int forge_group_destroy(forge_group* g);
int forge_group_size(forge_group* g, int32_t* count, int32_t* emulated);
int forge_group_stream(forge_group* g, int32_t rank, void** stream);
int forge_group_synchronize(forge_group* g);

/* mapreduce (primitives.hpp:348-351) of the concatenation of the shards
 * src[r][0..n[r]): local one-kernel mapreduce per shard, all-gather of the G
 * partials, rank-order fold on every device.  *result_host (nullable) gets the
 * S value (synchronous readback from rank 0); forge_sharded_result_dev gives
 * each shard's device copy. */
int forge_sharded_mapreduce(forge_group* g, forge_op op, const void* const* src, const uint64_t* n,
                            void* const* ws, const uint64_t* ws_bytes, void* result_host);
int forge_sharded_result_dev(forge_group* g, int32_t rank, void** value_dev);

/* scan (primitives.hpp:440-443) of the concatenation of the shards: dst[r]
 * receives shard r's slice of the global scan.  Reduce-then-scan: ordered shard
 * totals, all-gather, exclusive rank-order fold into a device carry, carry-
 * seeded single-pass scan.  ws_bytes[r] must cover both the PRIM_SCAN and the
 * PRIM_MAPREDUCE workspace of shard r (the shard total is reduced with it). */
int forge_sharded_scan(forge_group* g, forge_op op, int32_t inclusive, const void* const* src,
                       void* const* dst, const uint64_t* n, void* const* ws, const uint64_t* ws_bytes);

/* matvec / gevm (primitives.hpp:776-791) of a global n x p column-major A,
 * COLUMNS sharded: A_blocks[r] is shard r's n x p_r column block (p_r from
 * forge_shard_range(p_cols, r, G)), x[r] the full length-n x on shard r,
 * y_blocks[r] its p_r outputs.  No collective. */
int forge_sharded_matvec(forge_group* g, forge_op op, const void* const* A_blocks, uint64_t n,
                         uint64_t p_cols, const void* const* x, void* const* y_blocks, void* const* ws,
                         const uint64_t* ws_bytes);

/* vecmat / gemv (primitives.hpp:795-807), ROWS sharded: A_blocks[r] is shard
 * r's n_r x p row block, column-major with lda = n_r (n_r from
 * forge_shard_range(n, r, G)), x[r] the full length-p x, z_blocks[r] its n_r
 * outputs.  No collective. */
int forge_sharded_vecmat(forge_group* g, forge_op op, const void* const* A_blocks, uint64_t n,
                         uint64_t p_cols, const void* const* x, void* const* z_blocks, void* const* ws,
                         const uint64_t* ws_bytes);

/* scan over BLOCK-CYCLIC shards with a cross-GPU decoupled look-back
 * (the protocol of prim::scan, primitives.hpp:518-576,
 * extended across devices): the global array of n elements is cut into chunks
 * of chunk_elems (a positive multiple of forge_cyclic_chunk_quantum(op));
 * chunk c lives on shard c mod G, each shard holding its chunks back to back
 * (forge_cyclic_local_n elements).  Tile states live on their owner and are
 * read by the next shard over peer memory (NVLink / NVSwitch; peer access is
 * enabled on first use): no collective, 2n/G HBM bytes per GPU (reduce-then-
 * scan: 3n/G).  dst[r] receives shard r's elements of the global scan, same
 * layout.  ws_bytes[r] >= forge_cyclic_workspace_bytes(op, local_n).  Ops with
 * sizeof(S) == sizeof(T) <= 8 bytes; an emulated group needs
 * (chunk_elems / quantum) * G <= the SM count (one launch serves all shards). */
int forge_cyclic_chunk_quantum(forge_op op, uint64_t* elems);
int forge_cyclic_local_n(uint64_t n, uint64_t chunk_elems, int32_t rank, int32_t count, uint64_t* local_n);
int forge_cyclic_workspace_bytes(forge_op op, uint64_t local_n, uint64_t* bytes);
int forge_sharded_scan_cyclic(forge_group* g, forge_op op, int32_t inclusive, const void* const* src,
                              void* const* dst, uint64_t n, uint64_t chunk_elems, void* const* ws,
                              const uint64_t* ws_bytes);

#ifdef __cplusplus
}
#endif

#endif /* FORGE_H_ */
