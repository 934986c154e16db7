// capi.cu — the extern "C" surface of include/forge.h (core: machine, buffers,
// descriptors, workspaces, vcopy, synthetic data, copy).  The primitive entry
// points live in capi_scan.cu, capi_reduce.cu and capi_matrix.cu so the
// menu's kernel instantiations compile in parallel.
#include "capi_common.cuh"
#include "forge/litmus.hpp"

// ---------------------------------------------------------------------------
// Synthetic data on the device (bit-identical to oracle/oracle.c gen_one).

namespace {

__device__ __forceinline__ uint64_t dmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float dsym(uint64_t u) {
  return __fadd_rn(__fmul_rn(float(int32_t(u >> 40)), 0x1p-23f), -1.0f);
}
__device__ __forceinline__ float dpos(uint64_t u) { return __fmul_rn(float(int32_t(u >> 40)), 0x1p-24f); }
// variant 2: NaN (random payload and sign) / +-inf / signed zeros / small
// integers among ordinary values — oracle.c gen_f32_special, bit for bit.
__device__ __forceinline__ float dspecial(uint64_t u) {
  const uint32_t low = uint32_t(u & 0xFFFFu);
  if (low < 2u) return __uint_as_float(0x7fc00000u | uint32_t((u >> 16) & 0x3FFFFFu) | (low ? 0x80000000u : 0u));
  if (low < 4u) return __uint_as_float(low == 2u ? 0x7f800000u : 0xff800000u);
  if (low < 0x2000u) return __uint_as_float((u >> 16) & 1u ? 0x80000000u : 0u);
  if (low < 0x3000u) return __fadd_rn(float(int32_t((u >> 16) & 7u)), -4.0f);
  return dsym(u);
}

__global__ void fill_kernel(int op, unsigned char* dst, uint64_t n, uint64_t seed, uint64_t base,
                            int variant) {
  const uint64_t gs = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += gs) {
    const uint64_t idx = base + i;
    const uint64_t u = dmix(seed ^ idx);
    switch (op) {
      case FORGE_OP_F32_SUM: case FORGE_OP_F32_SUMSQ: case FORGE_OP_F32_MAX: case FORGE_OP_F32_MIN:
      case FORGE_OP_F32_LOGSUMEXP: case FORGE_OP_MV_F32_PLUS_TIMES: case FORGE_OP_MV_F32_MIN_PLUS:
      case FORGE_OP_MV_F32_MAX_PLUS:
        reinterpret_cast<float*>(dst)[i] = variant == 1 ? dpos(u) : variant == 2 ? dspecial(u) : dsym(u);
        break;
      case FORGE_OP_F64_SUM: case FORGE_OP_MV_F64_PLUS_TIMES:
        reinterpret_cast<double*>(dst)[i] = __dadd_rn(__dmul_rn(double(int64_t(u >> 11)), 0x1p-52), -1.0);
        break;
      case FORGE_OP_I32_SUM: case FORGE_OP_I32_MAX: case FORGE_OP_I32_MIN: case FORGE_OP_U32_SUM:
      case FORGE_OP_MV_I32_PLUS_TIMES: {
        uint32_t v = uint32_t(u >> 32);
        if (variant == 1) v &= 0xFFu;
        reinterpret_cast<uint32_t*>(dst)[i] = v;
        break;
      }
      case FORGE_OP_I64_SUM:
        reinterpret_cast<uint64_t*>(dst)[i] = u;
        break;
      case FORGE_OP_AFFINE_F32: {
        forge::alg::Affine v;
        v.a = __fadd_rn(1.0f, __fmul_rn(float(int32_t((u >> 50) & 0x3FFF) - 8192), 0x1p-23f));
        v.b = __fadd_rn(__fmul_rn(float(int32_t((u >> 8) & 0xFFFFFF)), 0x1p-23f), -1.0f);
        reinterpret_cast<forge::alg::Affine*>(dst)[i] = v;
        break;
      }
      case FORGE_OP_ARGMAX_F32I32: {
        forge::alg::ArgMax v;
        v.v = variant == 1 ? float(int32_t((u >> 60) & 0xF)) : variant == 2 ? dspecial(u) : dsym(u);
        v.i = int32_t(uint32_t(idx));
        reinterpret_cast<forge::alg::ArgMax*>(dst)[i] = v;
        break;
      }
      case FORGE_OP_MAT2_U32: case FORGE_OP_MV_MAT2_U32: {
        const uint64_t u2 = dmix(u);
        // odd diagonal, even off-diagonal (invertible mod 2^32; oracle.c gen_one)
        forge::alg::Mat2 v{{uint32_t(u) | 1u, uint32_t(u >> 32) & ~1u, uint32_t(u2) & ~1u, uint32_t(u2 >> 32) | 1u}};
        reinterpret_cast<forge::alg::Mat2*>(dst)[i] = v;
        break;
      }
      case FORGE_OP_QUAT_F32: {
        const uint64_t u2 = dmix(u);
        const float w = dsym(u), x = dsym(u << 24), y = dsym(u2), z = dsym(u2 << 24);
        const float s1 = __fadd_rn(__fmul_rn(w, w), __fmul_rn(x, x));
        const float s2 = __fadd_rn(s1, __fmul_rn(y, y));
        const float s3 = __fadd_rn(s2, __fmul_rn(z, z));
        const float r = __fsqrt_rn(s3 > 0x1p-20f ? s3 : 1.0f);
        reinterpret_cast<forge::alg::Quaternion*>(dst)[i] =
            forge::alg::Quaternion{__fdiv_rn(w, r), __fdiv_rn(x, r), __fdiv_rn(y, r), __fdiv_rn(z, r)};
        break;
      }
      case FORGE_OP_UF8_F32_SUM:
        dst[i] = (unsigned char)(u >> 56);
        break;
      default:
        break;
    }
  }
}

}  // namespace

extern "C" {

const char* forge_last_error(void) { return g_last_error.c_str(); }
int forge_abi_version(void) { return FORGE_ABI_VERSION; }

int forge_device_count(int* out) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  *out = e == cudaSuccess ? c : 0;
  if (e != cudaSuccess) {
    set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return FORGE_ERR_NO_DEVICE;
  }
  return FORGE_OK;
}

int forge_get_op_info(forge_op op, forge_op_info* out) {
  auto fill = [&](auto e, uint32_t binary) -> int {
    using E = decltype(e);
    out->t_size = sizeof(typename E::T);
    out->s_size = sizeof(typename E::S);
    out->commutative = e.commutative ? 1u : 0u;
    out->binary = binary;
    out->name = e.name;
    return FORGE_OK;
  };
  int rc = menu::visit1(op, [&](auto e) { return fill(e, 0); });
  if (rc == FORGE_ERR_UNSUPPORTED) rc = menu::visit2(op, [&](auto e) { return fill(e, 1); });
  if (rc == FORGE_ERR_UNSUPPORTED) set_error("unknown forge_op");
  return rc;
}

void forge_arch_params_default(forge_arch_params* out) {
  ArchParams a;
  out->warp_width = a.warp_width;
  out->mapreduce_blocks = a.mapreduce_blocks;
  out->threads_per_block = a.threads_per_block;
  out->nitem_scan = a.nitem_scan;
  out->nitem_copy = a.nitem_copy;
  out->lookback_window = a.lookback_window;
  out->matvec_wide_warp_cols = a.matvec_wide_warp_cols;
  out->matvec_wide_block_threads = a.matvec_wide_block_threads;
  out->matvec_wide_min_outputs = a.matvec_wide_min_outputs;
}

// ---- machine ---------------------------------------------------------------

int forge_machine_create(int device, forge_machine** out) {
  return guarded([&]() -> int {
    *out = nullptr;
    *out = new forge_machine{Machine(device)};
    return FORGE_OK;
  });
}

int forge_machine_destroy(forge_machine* m) {
  return guarded([&]() -> int {
    delete m;
    return FORGE_OK;
  });
}

int forge_machine_stream(forge_machine* m, void** s) {
  return guarded([&]() -> int {
    *s = reinterpret_cast<void*>(m->m.stream());
    return FORGE_OK;
  });
}

int forge_machine_synchronize(forge_machine* m) {
  return guarded([&]() -> int {
    m->m.synchronize();
    return FORGE_OK;
  });
}

int forge_create_buffer(forge_machine* m, const char* descriptor, uint64_t length,
                        uint32_t base_alignment, forge_buffer_id* out) {
  return guarded([&]() -> int {
    *out = m->m.create_buffer(parse_descriptor(descriptor ? descriptor : ""), length, base_alignment);
    return FORGE_OK;
  });
}

int forge_destroy_buffer(forge_machine* m, forge_buffer_id id) {
  return guarded([&]() -> int {
    m->m.destroy_buffer(id);
    return FORGE_OK;
  });
}

int forge_buffer_length(forge_machine* m, forge_buffer_id id, uint64_t* out) {
  return guarded([&]() -> int {
    *out = m->m.buffer_length(id);
    return FORGE_OK;
  });
}
int forge_buffer_elem_size(forge_machine* m, forge_buffer_id id, uint32_t* out) {
  return guarded([&]() -> int {
    *out = m->m.buffer_elem_size(id);
    return FORGE_OK;
  });
}
int forge_buffer_alignment(forge_machine* m, forge_buffer_id id, uint32_t* out) {
  return guarded([&]() -> int {
    *out = m->m.buffer_alignment(id);
    return FORGE_OK;
  });
}
int forge_buffer_device_ptr(forge_machine* m, forge_buffer_id id, void** out) {
  return guarded([&]() -> int {
    *out = m->m.device_ptr(id);
    return FORGE_OK;
  });
}

int forge_write_bytes(forge_machine* m, forge_buffer_id id, uint64_t elem_offset, const void* src,
                      uint64_t bytes) {
  return guarded([&]() -> int {
    m->m.write_bytes(id, elem_offset,
                     std::span<const std::byte>(static_cast<const std::byte*>(src), bytes));
    return FORGE_OK;
  });
}

int forge_read_bytes(forge_machine* m, forge_buffer_id id, uint64_t elem_offset, void* dst,
                     uint64_t bytes) {
  return guarded([&]() -> int {
    m->m.read_bytes(id, elem_offset, std::span<std::byte>(static_cast<std::byte*>(dst), bytes));
    return FORGE_OK;
  });
}

int forge_fill_zero(forge_machine* m, forge_buffer_id id) {
  return guarded([&]() -> int {
    m->m.fill_zero(id);
    return FORGE_OK;
  });
}

int forge_descriptor_info(const char* descriptor, uint32_t* size, uint32_t* alignment,
                          char* canonical, uint64_t cap) {
  return guarded([&]() -> int {
    TypeDescriptor d = parse_descriptor(descriptor ? descriptor : "");
    if (size) *size = d.size();
    if (alignment) *alignment = d.alignment();
    if (canonical && cap) {
      const std::string s = to_string(d);
      std::strncpy(canonical, s.c_str(), cap - 1);
      canonical[cap - 1] = 0;
    }
    return FORGE_OK;
  });
}

int forge_value_bytes_equal(const char* descriptor, const void* a, const void* b, int32_t* equal) {
  return guarded([&]() -> int {
    TypeDescriptor d = parse_descriptor(descriptor ? descriptor : "");
    *equal = value_bytes_equal(d, std::span<const std::byte>(static_cast<const std::byte*>(a), d.size()),
                               std::span<const std::byte>(static_cast<const std::byte*>(b), d.size()))
                 ? 1
                 : 0;
    return FORGE_OK;
  });
}

// ---- workspaces ------------------------------------------------------------

int forge_required_workspace(forge_primitive prim, uint32_t accum_size, uint64_t n, uint64_t p_cols,
                             const forge_arch_params* params, uint64_t* bytes) {
  return guarded([&]() -> int {
    *bytes = prim::required_workspace(static_cast<prim::Primitive>(prim), accum_size, n, p_cols,
                                      to_params(params));
    return FORGE_OK;
  });
}

int forge_make_scan_workspace(forge_machine* m, forge_op op, uint64_t n,
                              const forge_arch_params* params, forge_workspace* out) {
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) {
      using E = decltype(e);
      to_c(prim::make_scan_workspace<typename E::S>(m->m, n, to_params(params)), out);
      return FORGE_OK;
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "1-D") : rc;
  });
}

int forge_make_mapreduce_workspace(forge_machine* m, forge_op op, const forge_arch_params* params,
                                   forge_workspace* out) {
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) {
      using E = decltype(e);
      to_c(prim::make_mapreduce_workspace<typename E::S>(m->m, to_params(params)), out);
      return FORGE_OK;
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "1-D") : rc;
  });
}

int forge_make_mat_workspace(forge_machine* m, forge_op op, uint64_t reduce_len, uint64_t outputs,
                             const forge_arch_params* params, forge_workspace* out) {
  return guarded([&]() -> int {
    auto mk = [&](auto e) {
      using E = decltype(e);
      to_c(prim::make_mat_workspace<typename E::S>(m->m, reduce_len, outputs, to_params(params)), out);
      return FORGE_OK;
    };
    int rc = menu::visit2(op, mk);
    if (rc == FORGE_ERR_UNSUPPORTED) rc = menu::visit1(op, mk);
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "matrix") : rc;
  });
}

int forge_workspace_release(forge_machine* m, forge_workspace* ws) {
  return guarded([&]() -> int {
    Workspace w = from_c(ws);
    w.release(m->m);
    to_c(w, ws);
    return FORGE_OK;
  });
}

// ---- primitives ------------------------------------------------------------

int forge_set_mutation_flags(int32_t relax_scan_flag, int32_t relax_mapreduce_flag) {
  g_mutate.relax_scan_flag = relax_scan_flag != 0;
  g_mutate.relax_mapreduce_flag = relax_mapreduce_flag != 0;
  return FORGE_OK;
}

int forge_set_schedule_perturbation(uint64_t seed, uint32_t delay_ns) {
  g_perturb_seed = seed;
  g_perturb_ns = seed ? delay_ns : 0;
  return FORGE_OK;
}






int forge_mapreduce_2d(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                       forge_reduce_axis axis, forge_view out, forge_workspace* ws,
                       const forge_arch_params* params, forge_launch_report* report) {
  return guarded([&]() -> int {
    return axis == FORGE_AXIS_ROWS ? mapreduce_2d_rows(m, spec, A, n, p_cols, out, ws, params, report)
                                   : mapreduce_2d_cols(m, spec, A, n, p_cols, out, ws, params, report);
  });
}

int forge_vcopy(forge_machine* m, forge_view src, forge_view dst, uint32_t nitem,
                const forge_arch_params* params, forge_launch_report* report) {
  return guarded([&]() -> int {
    const uint32_t es = m->m.buffer_elem_size(src.buf);
    if (m->m.buffer_elem_size(dst.buf) != es)
      raise(ErrorCode::InvalidArgument, "vcopy: element sizes differ");
    ArchParams ap = to_params(params);
    LaunchReport r;
    switch (es) {
      case 1: r = prim::vcopy(m->m, view_of<uint8_t>(src), view_of<uint8_t>(dst), nitem, ap); break;
      case 2: r = prim::vcopy(m->m, view_of<uint16_t>(src), view_of<uint16_t>(dst), nitem, ap); break;
      case 4: r = prim::vcopy(m->m, view_of<uint32_t>(src), view_of<uint32_t>(dst), nitem, ap); break;
      case 8: r = prim::vcopy(m->m, view_of<uint64_t>(src), view_of<uint64_t>(dst), nitem, ap); break;
      case 16: r = prim::vcopy(m->m, view_of<alg::Mat2>(src), view_of<alg::Mat2>(dst), nitem, ap); break;
      default: {
        // Any other element size: contiguous byte copy of whole elements.
        if (src.stride != 1 || dst.stride != 1)
          raise(ErrorCode::Unsupported, "vcopy of strided views needs a 1/2/4/8/16-byte element");
        if (nitem != 1 && nitem != 2 && nitem != 4 && nitem != 8 && nitem != 16)
          raise(ErrorCode::InvalidNitem, "vcopy nitem");
        if (src.length != dst.length) raise(ErrorCode::DimensionMismatch, "vcopy lengths differ");
        (void)ap.normalized();
        const uint8_t* sp = static_cast<const uint8_t*>(m->m.device_ptr(src.buf)) + src.offset * es;
        uint8_t* dp = static_cast<uint8_t*>(m->m.device_ptr(dst.buf)) + dst.offset * es;
        if ((src.offset + src.length) > m->m.buffer_length(src.buf) ||
            (dst.offset + dst.length) > m->m.buffer_length(dst.buf))
          raise(ErrorCode::InvalidArgument, "view exceeds its buffer");
        const uint64_t bytes = src.length * es;
        r.buffers.resize(m->m.buffer_count());
        m->m.begin_timing();
        cudaError_t e = cuda::launch_vcopy<uint8_t>(sp, dp, bytes, m->m.stream());
        double secs = 0;
        cudaError_t e2 = m->m.end_timing(secs);
        r.ok = e == cudaSuccess && e2 == cudaSuccess;
        r.steps = 1;
        r.wall_seconds = secs;
        if (!r.ok) {
          r.fault.kind = FaultKind::Internal;
          r.fault.detail = cudaGetErrorString(e != cudaSuccess ? e : e2);
        }
      }
    }
    return finish(r, report);
  });
}

int forge_vload_pattern(uint64_t offset, uint32_t nitem, uint32_t* segs, uint32_t* count) {
  return guarded([&]() -> int {
    intr::LoadPattern p = intr::vload_pattern(offset, nitem);
    for (uint32_t i = 0; i < p.count; ++i) segs[i] = p.seg[i];
    *count = p.count;
    return FORGE_OK;
  });
}

// ---- litmus (forge::lit) -------------------------------------------------------

int forge_litmus_parse(const char* spec_text) {
  return guarded([&]() -> int {
    if (!spec_text) raise(ErrorCode::InvalidArgument, "litmus: null text");
    (void)lit::parse_litmus(spec_text);
    return FORGE_OK;
  });
}

int forge_litmus_run(const char* spec_text, uint64_t seed_begin, uint64_t seed_end, forge_litmus_result* out,
                     char* histogram, uint64_t histogram_cap) {
  return guarded([&]() -> int {
    if (!spec_text || !out) raise(ErrorCode::InvalidArgument, "litmus: null argument");
    const lit::LitmusSpec spec = lit::parse_litmus(spec_text);
    const lit::LitmusResult r = lit::run_litmus(spec, seed_begin, seed_end);
    out->seeds_run = r.seeds_run;
    out->assert_violations = r.assert_violations;
    out->faults = r.faults;
    out->distinct_outcomes = r.histogram.size();
    if (histogram && histogram_cap > 0) {
      std::vector<std::pair<uint64_t, std::string>> rows;
      for (const auto& [o, c] : r.histogram) rows.emplace_back(c, o.to_string());
      std::stable_sort(rows.begin(), rows.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
      std::string text;
      for (const auto& [c, o] : rows) text += std::to_string(c) + "\t" + o + "\n";
      const size_t n = std::min<size_t>(text.size(), size_t(histogram_cap - 1));
      std::memcpy(histogram, text.data(), n);
      histogram[n] = 0;
    }
    if (r.faults) {
      set_error("litmus: " + r.first_fault.detail);
      return FORGE_ERR_DEVICE_FAULT;
    }
    return FORGE_OK;
  });
}

// ---- device-pointer layer ---------------------------------------------------

int forge_dev_workspace_bytes(forge_primitive prim, forge_op op, uint64_t n, uint64_t p_cols,
                              uint64_t* bytes) {
  return guarded([&]() -> int {
    int rc = FORGE_ERR_UNSUPPORTED;
    switch (prim) {
      case FORGE_PRIM_SCAN:
        rc = menu::visit1(op, [&](auto e) {
          using E = decltype(e);
          *bytes = cuda::ScanWs<typename E::T, typename E::S, typename E::Op>::bytes(n);
          return FORGE_OK;
        });
        break;
      case FORGE_PRIM_MAPREDUCE:
        rc = menu::visit1(op, [&](auto e) {
          using E = decltype(e);
          // commutative mapreduce and the ordered reduce share one workspace
          *bytes = std::max<uint64_t>(
              cuda::MapReduceWs<typename E::S>::bytes(cuda::mapreduce_max_grid()),
              cuda::OrderedReduceWs<typename E::S, typename E::Op>::bytes(cuda::mapreduce_max_grid()));
          return FORGE_OK;
        });
        break;
      case FORGE_PRIM_MATVEC:
        rc = menu::visit2(op, [&](auto e) {
          using E = decltype(e);
          *bytes = cuda::gevm_ws_bytes<typename E::T, typename E::S>(n, p_cols);
          return FORGE_OK;
        });
        break;
      case FORGE_PRIM_VECMAT:
        rc = menu::visit2(op, [&](auto e) {
          using E = decltype(e);
          *bytes = cuda::gemv_ws_bytes<typename E::T, typename E::S>(n, p_cols);
          return FORGE_OK;
        });
        break;
      default:
        *bytes = 0;
        rc = FORGE_OK;
    }
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "device") : rc;
  });
}







int forge_dev_copy(const void* src, void* dst, uint64_t bytes, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_copy");
  return guarded([&]() -> int {
    auto st = static_cast<cudaStream_t>(stream);
    if (bytes % 4 == 0 && cuda::is_aligned(src, 4) && cuda::is_aligned(dst, 4))
      return from_cuda(cuda::launch_vcopy<uint32_t>(static_cast<const uint32_t*>(src),
                                                    static_cast<uint32_t*>(dst), bytes / 4, st),
                       "copy launch");
    return from_cuda(cuda::launch_vcopy<uint8_t>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst),
                                                 bytes, st),
                     "copy launch");
  });
}

int forge_dev_fill_synthetic(forge_op op, void* dst, uint64_t n, uint64_t seed, uint64_t index_base,
                             int32_t variant, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_fill_synthetic");
  return guarded([&]() -> int {
    if (n == 0) return FORGE_OK;
    uint64_t grid = (n + 255) / 256;
    const uint64_t cap = uint64_t(cuda::device_props().sm_count) * 16;
    if (grid > cap) grid = cap;
    fill_kernel<<<uint32_t(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        int(op), static_cast<unsigned char*>(dst), n, seed, index_base, variant);
    return from_cuda(cudaGetLastError(), "fill launch");
  });
}

#ifdef FORGE_DEV
// Development build only (make DEV=1): the per-tile phase trace of the last
// scan run with FORGE_SCAN_TRACE=1 (tools/trace_scan.py), 8 words per tile.
int forge_dev_scan_trace(void** ptr, uint64_t* words) {
  *ptr = cuda::scan_trace_buffer();
  *words = cuda::scan_trace_words();
  return FORGE_OK;
}
#endif

}  // extern "C"
