// capi_mr2d_rows.cu — mapreduce_2d (primitives.hpp:809-836), axis Rows: one value per column, the unary map lifted into matvec
// (a translation unit of its own: the menu's kernel instantiations compile in parallel).
#include "capi_common.cuh"

namespace forge::capi {

int mapreduce_2d_rows(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                     forge_view out, forge_workspace* ws, const forge_arch_params* params,
                     forge_launch_report* report) {
  Workspace w = from_c(ws);
  int rc = menu::visit1(spec.op, [&](auto e) {
    using E = decltype(e);
    using T = typename E::T;
    using S = typename E::S;
    const auto s1 = e.spec(spec.has_identity != 0);
    prim::SemiringSpec<prim::detail::LiftSecond<typename E::F>, S, typename E::Op> lifted{
        {s1.map}, s1.op, s1.identity, s1.commutative};
    const intr::View<T> none{A.buf, 0, 0, 1};
    LaunchReport r = prim::matvec<T, S>(m->m, lifted, view_of<T>(A), n, p_cols, none, view_of<S>(out), w,
                                       to_params(params), {}, /*uses_vector=*/false);
    return finish(r, report);
  });
  return rc == FORGE_ERR_UNSUPPORTED ? unsupported_op(spec.op, "mapreduce_2d") : rc;
}

}  // namespace forge::capi
