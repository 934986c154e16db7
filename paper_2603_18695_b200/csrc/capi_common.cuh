// capi_common.cuh — shared helpers of the C-ABI translation units (capi*.cu):
// together they are the extern "C" surface of include/forge.h over the
// forge::prim templates and the sm_100a kernels (the `capi.cpp` that
// /root/reference/proj/src/CMakeLists.txt:13-17 declares but never ships).
//
// Every entry point: exceptions never cross the boundary.  forge::Error ->
// 1 + ErrorCode; forge::NoDeviceError -> FORGE_ERR_NO_DEVICE; a CUDA failure
// -> FORGE_ERR_DEVICE_FAULT (and LaunchReport{ok = 0} when a report is passed).
#pragma once

#include <cstring>
#include <string>

#include "forge.h"
#include "forge/bitstype.hpp"
#include "menu.cuh"

using namespace forge;
using forge::prim::ArchParams;
using forge::prim::Workspace;

namespace forge::capi {

inline thread_local std::string g_last_error;
inline thread_local prim::MutationFlags g_mutate;  // forge_set_mutation_flags (test-only ablation)
inline thread_local uint64_t g_perturb_seed = 0;   // forge_set_schedule_perturbation (test only)
inline thread_local uint32_t g_perturb_ns = 0;

inline cuda::ScanTestHooks scan_hooks() {
  return cuda::ScanTestHooks{g_mutate.relax_scan_flag, g_perturb_seed, g_perturb_ns};
}

inline void set_error(const std::string& s) { g_last_error = s; }

template <class Fn>
inline int guarded(Fn&& fn) {
  try {
    const int rc = fn();
    if (rc == FORGE_OK) g_last_error.clear();
    return rc;
  } catch (const forge::Error& e) {
    set_error(std::string(to_string(e.code())) + ": " + e.what());
    return e.status();
  } catch (const forge::NoDeviceError& e) {
    set_error(e.what());
    return FORGE_ERR_NO_DEVICE;
  } catch (const std::exception& e) {
    set_error(e.what());
    return FORGE_ERR_DEVICE_FAULT;
  }
}

inline int unsupported_op(forge_op op, const char* what) {
  set_error(std::string("Unsupported: op ") + std::to_string(int(op)) + " is not in the " + what +
            " menu");
  return FORGE_ERR_UNSUPPORTED;
}

inline ArchParams to_params(const forge_arch_params* p) {
  ArchParams a;
  if (p) {
    a.warp_width = p->warp_width;
    a.mapreduce_blocks = p->mapreduce_blocks;
    a.threads_per_block = p->threads_per_block;
    a.nitem_scan = p->nitem_scan;
    a.nitem_copy = p->nitem_copy;
    a.lookback_window = p->lookback_window;
    a.matvec_wide_warp_cols = p->matvec_wide_warp_cols;
    a.matvec_wide_block_threads = p->matvec_wide_block_threads;
    a.matvec_wide_min_outputs = p->matvec_wide_min_outputs;
  }
  return a;
}

inline Workspace from_c(const forge_workspace* w) {
  Workspace r;
  if (!w) return r;
  r.tile_aggregate = w->tile_aggregate;
  r.tile_prefix = w->tile_prefix;
  r.tile_flag = w->tile_flag;
  r.partials = w->partials;
  r.flags = w->flags;
  r.result = w->result;
  r.tiles = w->tiles;
  r.slots = w->slots;
  return r;
}

inline void to_c(const Workspace& r, forge_workspace* w) {
  w->tile_aggregate = r.tile_aggregate;
  w->tile_prefix = r.tile_prefix;
  w->tile_flag = r.tile_flag;
  w->partials = r.partials;
  w->flags = r.flags;
  w->result = r.result;
  w->tiles = r.tiles;
  w->slots = r.slots;
}

inline int finish(const LaunchReport& r, forge_launch_report* out) {
  if (out) {
    out->ok = r.ok ? 1 : 0;
    out->fault_kind = int32_t(r.fault.kind);
    out->steps = r.steps;
    out->wall_seconds = r.wall_seconds;
    std::memset(out->detail, 0, sizeof(out->detail));
    std::strncpy(out->detail, r.fault.detail.c_str(), sizeof(out->detail) - 1);
  }
  if (!r.ok) {
    set_error("device fault: " + r.fault.detail);
    return FORGE_ERR_DEVICE_FAULT;
  }
  return FORGE_OK;
}

template <class T>
inline intr::View<T> view_of(const forge_view& v) {
  return intr::View<T>{v.buf, v.offset, v.length, v.stride == 0 ? 1 : v.stride};
}

inline int from_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FORGE_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FORGE_ERR_DEVICE_FAULT;
}

inline int require_ws(uint64_t have, uint64_t need, const char* what) {
  if (have < need) {
    set_error(std::string("WorkspaceTooSmall: ") + what + " needs " + std::to_string(need) +
              " bytes, got " + std::to_string(have));
    return FORGE_ERR_WORKSPACE_TOO_SMALL;
  }
  return FORGE_OK;
}

}  // namespace forge::capi

struct forge_machine {
  Machine m;
};

namespace forge::capi {
// mapreduce_2d by axis (capi_mr2d_rows.cu / capi_mr2d_cols.cu)
int mapreduce_2d_rows(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                      forge_view out, forge_workspace* ws, const forge_arch_params* params,
                      forge_launch_report* report);
int mapreduce_2d_cols(forge_machine* m, forge_semiring spec, forge_view A, uint64_t n, uint64_t p_cols,
                      forge_view out, forge_workspace* ws, const forge_arch_params* params,
                      forge_launch_report* report);
}  // namespace forge::capi

using namespace forge::capi;
