// capi_scan.cu — C-ABI entry points: scan (include/forge.h).
#include "capi_common.cuh"

extern "C" {

int forge_scan(forge_machine* m, forge_semiring spec, forge_view src, forge_view dst,
               int32_t inclusive, forge_workspace* ws, const forge_arch_params* params,
               forge_launch_report* report) {
  return guarded([&]() -> int {
    Workspace w = from_c(ws);
    int rc = menu::visit1(spec.op, [&](auto e) {
      using E = decltype(e);
      prim::RunOptions ro;
      ro.mutate = g_mutate;
      ro.schedule.seed = g_perturb_seed;
      LaunchReport r = prim::scan(m->m, e.spec(spec.has_identity != 0), view_of<typename E::T>(src),
                                  view_of<typename E::S>(dst), inclusive != 0, w, to_params(params), ro);
      return finish(r, report);
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(spec.op, "scan") : rc;
  });
}

int forge_dev_scan(forge_op op, int32_t inclusive, const void* src, void* dst, uint64_t n,
                   const void* carry_in_dev, void* total_out_dev, void* ws, uint64_t ws_bytes,
                   void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_scan");
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      if (n == 0) return FORGE_OK;
      using WsT = cuda::ScanWs<T, S, typename E::Op>;
      int w = require_ws(ws_bytes, WsT::min_bytes_for(cuda::ceil_div(n, WsT::kTileGeneral)), "scan");
      if (w) return w;
      return from_cuda(cuda::launch_scan<T, S>(static_cast<const T*>(src), 1, static_cast<S*>(dst), 1, n,
                                               inclusive != 0, typename E::F{}, typename E::Op{}, e.identity,
                                               static_cast<const S*>(carry_in_dev),
                                               static_cast<S*>(total_out_dev), ws, ws_bytes,
                                               static_cast<cudaStream_t>(stream), scan_hooks()),
                       "scan launch");
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "scan") : rc;
  });
}

}  // extern "C"
