// capi_matrix.cu — C-ABI entry points: matvec, vecmat and mapreduce_2d (include/forge.h).
#include "capi_common.cuh"

extern "C" {

int forge_matvec(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                 forge_view x, forge_view y, forge_workspace* ws, const forge_arch_params* params,
                 forge_launch_report* report, int32_t uses_vector) {
  return guarded([&]() -> int {
    Workspace w = from_c(ws);
    int rc = menu::visit2(spec.op, [&](auto e) {
      using E = decltype(e);
      LaunchReport r = prim::matvec<typename E::T, typename E::S>(
          m->m, e.spec(spec.has_identity != 0), view_of<typename E::T>(A), n, p_cols,
          view_of<typename E::T>(x), view_of<typename E::S>(y), w, to_params(params), {}, uses_vector != 0);
      return finish(r, report);
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(spec.op, "matrix") : rc;
  });
}

int forge_vecmat(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                 forge_view x, forge_view z, forge_workspace* ws, const forge_arch_params* params,
                 forge_launch_report* report, int32_t uses_vector) {
  return guarded([&]() -> int {
    Workspace w = from_c(ws);
    int rc = menu::visit2(spec.op, [&](auto e) {
      using E = decltype(e);
      LaunchReport r = prim::vecmat<typename E::T, typename E::S>(
          m->m, e.spec(spec.has_identity != 0), view_of<typename E::T>(A), n, p_cols,
          view_of<typename E::T>(x), view_of<typename E::S>(z), w, to_params(params), {}, uses_vector != 0);
      return finish(r, report);
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(spec.op, "matrix") : rc;
  });
}

int forge_dev_matvec_lda(forge_op op, const void* A, uint64_t n, uint64_t p_cols, uint64_t lda, const void* x,
                         void* y, void* ws, uint64_t ws_bytes, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_matvec");
  return guarded([&]() -> int {
    if (lda != 0 && lda < n) raise(ErrorCode::InvalidArgument, "matvec: lda < n");
    int rc = menu::visit2(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      int w = require_ws(ws_bytes, cuda::gevm_ws_bytes<T, S>(n, p_cols), "matvec");
      if (w) return w;
      auto st = static_cast<cudaStream_t>(stream);
      cudaError_t err =
          e.commutative
              ? cuda::launch_gevm<T, S, typename E::F, typename E::Op, true, false>(
                    static_cast<const T*>(A), n, p_cols, static_cast<const T*>(x), static_cast<S*>(y),
                    typename E::F{}, typename E::Op{}, ws, st, lda)
              : cuda::launch_gevm<T, S, typename E::F, typename E::Op, true, true>(
                    static_cast<const T*>(A), n, p_cols, static_cast<const T*>(x), static_cast<S*>(y),
                    typename E::F{}, typename E::Op{}, ws, st, lda);
      return from_cuda(err, "matvec launch");
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "matrix") : rc;
  });
}

int forge_dev_matvec(forge_op op, const void* A, uint64_t n, uint64_t p_cols, const void* x, void* y,
                     void* ws, uint64_t ws_bytes, void* stream) {
  return forge_dev_matvec_lda(op, A, n, p_cols, n, x, y, ws, ws_bytes, stream);
}

int forge_dev_vecmat_lda(forge_op op, const void* A, uint64_t n, uint64_t p_cols, uint64_t lda, const void* x,
                         void* z, void* ws, uint64_t ws_bytes, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_vecmat");
  return guarded([&]() -> int {
    if (lda != 0 && lda < n) raise(ErrorCode::InvalidArgument, "vecmat: lda < n");
    int rc = menu::visit2(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      int w = require_ws(ws_bytes, cuda::gemv_ws_bytes<T, S>(n, p_cols), "vecmat");
      if (w) return w;
      return from_cuda(cuda::launch_gemv<T, S, typename E::F, typename E::Op, true>(
                           static_cast<const T*>(A), n, p_cols, static_cast<const T*>(x), static_cast<S*>(z),
                           typename E::F{}, typename E::Op{}, ws, static_cast<cudaStream_t>(stream), lda),
                       "vecmat launch");
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "matrix") : rc;
  });
}

int forge_dev_vecmat(forge_op op, const void* A, uint64_t n, uint64_t p_cols, const void* x, void* z,
                     void* ws, uint64_t ws_bytes, void* stream) {
  return forge_dev_vecmat_lda(op, A, n, p_cols, n, x, z, ws, ws_bytes, stream);
}

}  // extern "C"
