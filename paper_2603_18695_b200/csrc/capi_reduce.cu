// capi_reduce.cu — C-ABI entry points: mapreduce, ordered reduce and the rank-order fold (include/forge.h).
#include "capi_common.cuh"

extern "C" {

int forge_mapreduce(forge_machine* m, forge_semiring spec, forge_view src, forge_workspace* ws,
                    const forge_arch_params* params, void* out_host, forge_launch_report* report) {
  return guarded([&]() -> int {
    Workspace w = from_c(ws);
    int rc = menu::visit1(spec.op, [&](auto e) {
      using E = decltype(e);
      typename E::S r{};
      LaunchReport rep = prim::mapreduce(m->m, e.spec(spec.has_identity != 0), view_of<typename E::T>(src), w,
                                         to_params(params), &r);
      if (rep.ok) std::memcpy(out_host, &r, sizeof(r));
      return finish(rep, report);
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(spec.op, "mapreduce") : rc;
  });
}

int forge_dev_mapreduce(forge_op op, const void* src, uint64_t n, void* out_dev, void* ws,
                        uint64_t ws_bytes, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_mapreduce");
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      if (!e.commutative) {
        set_error("InvalidArgument: mapreduce requires a commutative op; use forge_dev_reduce_ordered");
        return FORGE_ERR_INVALID_ARGUMENT;
      }
      if (n == 0)
        return from_cuda(cudaMemcpyAsync(out_dev, &e.identity, sizeof(S), cudaMemcpyHostToDevice, st),
                         "identity copy");
      int w = require_ws(ws_bytes, cuda::MapReduceWs<S>::bytes(cuda::mapreduce_max_grid()), "mapreduce");
      if (w) return w;
      return from_cuda(cuda::launch_mapreduce<T, S>(static_cast<const T*>(src), n, 1, typename E::F{},
                                                    typename E::Op{}, static_cast<S*>(out_dev), nullptr,
                                                    ws, st),
                       "mapreduce launch");
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "mapreduce") : rc;
  });
}

int forge_dev_reduce_ordered(forge_op op, const void* src, uint64_t n, void* out_dev, void* ws,
                             uint64_t ws_bytes, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_reduce_ordered");
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      if (n == 0)
        return from_cuda(cudaMemcpyAsync(out_dev, &e.identity, sizeof(S), cudaMemcpyHostToDevice, st),
                         "identity copy");
      int w = require_ws(ws_bytes, cuda::OrderedReduceWs<S, typename E::Op>::bytes(cuda::mapreduce_max_grid()),
                         "reduce_ordered");
      if (w) return w;
      return from_cuda(cuda::launch_reduce_ordered<T, S>(static_cast<const T*>(src), n, 1, typename E::F{},
                                                         typename E::Op{}, static_cast<S*>(out_dev), nullptr,
                                                         ws, st),
                       "reduce_ordered launch");
    });
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "reduce") : rc;
  });
}

int forge_dev_fold(forge_op op, const void* values_dev, uint32_t count, int32_t exclusive_upto,
                   void* out_dev, int32_t* has_out_dev, void* stream) {
  forge::prim::detail::NvtxRange nvtx_range("forge_dev_fold");
  return guarded([&]() -> int {
    auto go = [&](auto e) -> int {
      using E = decltype(e);
      using S = typename E::S;
      return from_cuda(cuda::launch_fold<S>(static_cast<const S*>(values_dev), count, exclusive_upto,
                                            typename E::Op{}, static_cast<S*>(out_dev), has_out_dev,
                                            static_cast<cudaStream_t>(stream)),
                       "fold launch");
    };
    int rc = menu::visit1(op, go);
    if (rc == FORGE_ERR_UNSUPPORTED) rc = menu::visit2(op, go);
    return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(op, "fold") : rc;
  });
}

}  // extern "C"
