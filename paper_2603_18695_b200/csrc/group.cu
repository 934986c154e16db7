// group.cu — single-process multi-GPU sharding behind the C-ABI (include/forge.h
// forge_group_* / forge_sharded_*): SURVEY.md §8(e) for C and C++ callers,
// without torch.  One shard per device, rank order = the order of the device
// list; the exchange is NCCL over NVLink / NVSwitch (ncclCommInitAll clique,
// libnccl.so.2 opened at first use so the library itself does not depend on
// NCCL), or — when every entry of the device list names the same GPU — device
// copies on that GPU: the EMULATED group, which runs the identical exchange
// logic with G shards on one B200 (the test harness of a 1-GPU box).
//
//   mapreduce  local one-kernel mapreduce per shard -> all-gather of the G
//              partials (sizeof(S) each) -> rank-order fold on every device;
//              the value is returned to the host from rank 0 (the reference's
//              `S* out`, primitives.hpp:425-429).
//   scan       reduce-then-scan: order-preserving shard totals -> all-gather ->
//              exclusive rank-order fold into a device carry -> single-pass scan
//              seeded with it (primitives.hpp:440-603 semantics over the
//              concatenation of the shards).  No host synchronisation between
//              the steps.
//   matvec     (gevm, primitives.hpp:776-791) columns sharded: shard r holds the
//              n x p_r column block (contiguous in column-major), x replicated.
//   vecmat     (gemv, :795-807) rows sharded: shard r holds the n_r x p row
//              block (column-major, lda = n_r), x replicated.  No collective.
//   scan_cyclic  block-cyclic chunks with a cross-GPU decoupled look-back over
//              peer memory (forge/cuda/scan_cyclic.cuh): 2n/G bytes per GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_common.cuh"
#include "forge/cuda/scan_cyclic.cuh"

using namespace forge::capi;

namespace {

// ---- NCCL, resolved at run time ------------------------------------------------
struct Nccl {
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string why;
  bool ok() const { return comm_init_all != nullptr; }
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      r.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return r;
    }
    r.comm_init_all = reinterpret_cast<decltype(r.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!r.comm_init_all || !r.comm_destroy || !r.all_gather || !r.group_start || !r.group_end ||
        !r.error_string) {
      r = Nccl{};
      r.why = "libnccl.so.2 lacks an expected symbol";
    }
    return r;
  }();
  return n;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FORGE_OK;
  set_error(std::string(what) + ": " + nccl().error_string(r));
  return FORGE_ERR_DEVICE_FAULT;
}

// Per-shard exchange scratch: one S value, the gathered G values, the carry
// and its has-flag.  S <= 16 bytes for every menu op.
constexpr uint64_t kSlot = 16;

struct Shard {
  int device = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  unsigned char* scratch = nullptr;  // [kSlot local | kSlot carry | 16 has | G * kSlot gathered]
  unsigned char* local() const { return scratch; }
  unsigned char* carry() const { return scratch + kSlot; }
  int32_t* has() const { return reinterpret_cast<int32_t*>(scratch + 2 * kSlot); }
  unsigned char* gathered() const { return scratch + 3 * kSlot; }
};

struct DeviceGuard {
  int saved = 0;
  DeviceGuard() { cudaGetDevice(&saved); }
  ~DeviceGuard() { cudaSetDevice(saved); }
};

}  // namespace

struct forge_group {
  std::vector<Shard> shards;
  bool emulated = false;  // every shard on the same device; exchange by device copies
  int size() const { return int(shards.size()); }
};

namespace {

int check_group(forge_group* g) {
  if (!g || g->shards.empty()) {
    set_error("InvalidArgument: null or empty forge_group");
    return FORGE_ERR_INVALID_ARGUMENT;
  }
  return FORGE_OK;
}

int use(const Shard& s) { return from_cuda(cudaSetDevice(s.device), "cudaSetDevice"); }

// All-gather of `bytes` from every shard's local() into every shard's
// gathered() (rank order).  Stream-ordered on each shard's stream.
int all_gather(forge_group* g, uint64_t bytes) {
  const int G = g->size();
  if (g->emulated) {
    // one device: shard r's slot r of every gathered buffer.  Each shard's
    // stream first waits for every other shard's local value.
    std::vector<cudaEvent_t> ev(G);
    for (int r = 0; r < G; ++r) {
      if (int rc = from_cuda(cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming), "event"); rc) return rc;
      if (int rc = from_cuda(cudaEventRecord(ev[r], g->shards[r].stream), "event record"); rc) return rc;
    }
    for (int d = 0; d < G; ++d) {
      const Shard& dst = g->shards[d];
      for (int r = 0; r < G; ++r) {
        if (int rc = from_cuda(cudaStreamWaitEvent(dst.stream, ev[r], 0), "stream wait"); rc) return rc;
        if (int rc = from_cuda(cudaMemcpyAsync(dst.gathered() + r * bytes, g->shards[r].local(), bytes,
                                               cudaMemcpyDeviceToDevice, dst.stream),
                               "gather copy");
            rc)
          return rc;
      }
    }
    // the next use of any local() slot is ordered after every copy out of it
    std::vector<cudaEvent_t> done(G);
    for (int d = 0; d < G; ++d) {
      cudaEventCreateWithFlags(&done[d], cudaEventDisableTiming);
      cudaEventRecord(done[d], g->shards[d].stream);
    }
    for (int r = 0; r < G; ++r)
      for (int d = 0; d < G; ++d) cudaStreamWaitEvent(g->shards[r].stream, done[d], 0);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : done) cudaEventDestroy(e);
    return FORGE_OK;
  }
  const Nccl& n = nccl();
  if (int rc = nccl_check(n.group_start(), "ncclGroupStart"); rc) return rc;
  for (const Shard& s : g->shards) {
    const ncclResult_t r = n.all_gather(s.local(), s.gathered(), bytes, ncclUint8, s.comm, s.stream);
    if (r != ncclSuccess) {
      n.group_end();
      return nccl_check(r, "ncclAllGather");
    }
  }
  return nccl_check(n.group_end(), "ncclGroupEnd");
}

int s_size_of(forge_op op, uint32_t* ss) {
  forge_op_info info{};
  if (int rc = forge_get_op_info(op, &info); rc) return rc;
  if (info.s_size > kSlot) {
    set_error("Unsupported: S larger than 16 bytes in the sharded exchange");
    return FORGE_ERR_UNSUPPORTED;
  }
  *ss = info.s_size;
  return FORGE_OK;
}

}  // namespace

extern "C" {

int forge_shard_range(uint64_t total, int32_t rank, int32_t count, uint64_t* lo, uint64_t* hi) {
  return guarded([&]() -> int {
    if (count <= 0 || rank < 0 || rank >= count || !lo || !hi) {
      set_error("InvalidArgument: forge_shard_range needs 0 <= rank < count");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    // shard r = [total*r/G, total*(r+1)/G), 128-bit products (no overflow)
    *lo = uint64_t((unsigned __int128)total * uint64_t(rank) / uint64_t(count));
    *hi = uint64_t((unsigned __int128)total * uint64_t(rank + 1) / uint64_t(count));
    return FORGE_OK;
  });
}

int forge_group_create(const int32_t* devices, int32_t count, forge_group** out) {
  return guarded([&]() -> int {
    if (!devices || count <= 0 || !out) {
      set_error("InvalidArgument: forge_group_create needs count >= 1 devices");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      set_error("no CUDA device: the library never falls back to the CPU");
      return FORGE_ERR_NO_DEVICE;
    }
    bool all_same = true, distinct = true;
    for (int i = 0; i < count; ++i) {
      if (devices[i] < 0 || devices[i] >= ndev) {
        set_error("InvalidArgument: device ordinal out of range");
        return FORGE_ERR_INVALID_ARGUMENT;
      }
      all_same &= devices[i] == devices[0];
      for (int j = 0; j < i; ++j) distinct &= devices[j] != devices[i];
    }
    if (count > 1 && !all_same && !distinct) {
      set_error("InvalidArgument: a group's devices are all distinct (NCCL) or all the same (emulated)");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    DeviceGuard guard;
    auto g = std::make_unique<forge_group>();
    g->emulated = count > 1 && all_same;
    g->shards.resize(count);
    for (int i = 0; i < count; ++i) {
      Shard& s = g->shards[i];
      s.device = devices[i];
      if (int rc = use(s); rc) return rc;
      if (int rc = from_cuda(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream"); rc) return rc;
      if (int rc = from_cuda(cudaMalloc(&s.scratch, 3 * kSlot + uint64_t(count) * kSlot), "scratch"); rc)
        return rc;
    }
    if (!g->emulated) {
      const Nccl& n = nccl();
      if (!n.ok()) {
        set_error("Unsupported: " + n.why);
        return FORGE_ERR_UNSUPPORTED;
      }
      std::vector<ncclComm_t> comms(count);
      std::vector<int> devs(devices, devices + count);
      if (int rc = nccl_check(n.comm_init_all(comms.data(), count, devs.data()), "ncclCommInitAll"); rc) return rc;
      for (int i = 0; i < count; ++i) g->shards[i].comm = comms[i];
    }
    *out = g.release();
    return FORGE_OK;
  });
}

int forge_group_destroy(forge_group* g) {
  return guarded([&]() -> int {
    if (!g) return FORGE_OK;
    DeviceGuard guard;
    for (Shard& s : g->shards) {
      cudaSetDevice(s.device);
      if (s.stream) cudaStreamSynchronize(s.stream);
      if (s.comm) nccl().comm_destroy(s.comm);
      if (s.scratch) cudaFree(s.scratch);
      if (s.stream) cudaStreamDestroy(s.stream);
    }
    delete g;
    return FORGE_OK;
  });
}

int forge_group_size(forge_group* g, int32_t* count, int32_t* emulated) {
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    if (count) *count = g->size();
    if (emulated) *emulated = g->emulated ? 1 : 0;
    return FORGE_OK;
  });
}

int forge_group_stream(forge_group* g, int32_t rank, void** stream) {
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    if (rank < 0 || rank >= g->size() || !stream) {
      set_error("InvalidArgument: rank out of range");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    *stream = g->shards[rank].stream;
    return FORGE_OK;
  });
}

int forge_group_synchronize(forge_group* g) {
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    DeviceGuard guard;
    for (const Shard& s : g->shards) {
      if (int rc = use(s); rc) return rc;
      if (int rc = from_cuda(cudaStreamSynchronize(s.stream), "group synchronize"); rc) return rc;
    }
    return FORGE_OK;
  });
}

int forge_sharded_mapreduce(forge_group* g, forge_op op, const void* const* src, const uint64_t* n,
                            void* const* ws, const uint64_t* ws_bytes, void* result_host) {
  forge::prim::detail::NvtxRange nvtx_range("forge_sharded_mapreduce");
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    uint32_t ss = 0;
    if (int rc = s_size_of(op, &ss); rc) return rc;
    DeviceGuard guard;
    const int G = g->size();
    for (int r = 0; r < G; ++r) {
      const Shard& s = g->shards[r];
      if (int rc = use(s); rc) return rc;
      if (int rc = forge_dev_mapreduce(op, src[r], n[r], s.local(), ws[r], ws_bytes[r], s.stream); rc) return rc;
    }
    if (G > 1) {
      if (int rc = all_gather(g, ss); rc) return rc;
      for (int r = 0; r < G; ++r) {
        const Shard& s = g->shards[r];
        if (int rc = use(s); rc) return rc;
        if (int rc = forge_dev_fold(op, s.gathered(), uint32_t(G), -1, s.local(), nullptr, s.stream); rc) return rc;
      }
    }
    if (result_host) {
      const Shard& s0 = g->shards[0];
      if (int rc = use(s0); rc) return rc;
      if (int rc = from_cuda(cudaMemcpyAsync(result_host, s0.local(), ss, cudaMemcpyDeviceToHost, s0.stream),
                             "result readback");
          rc)
        return rc;
      if (int rc = from_cuda(cudaStreamSynchronize(s0.stream), "result readback"); rc) return rc;
    }
    return FORGE_OK;
  });
}

int forge_sharded_result_dev(forge_group* g, int32_t rank, void** value_dev) {
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    if (rank < 0 || rank >= g->size() || !value_dev) {
      set_error("InvalidArgument: rank out of range");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    *value_dev = g->shards[rank].local();
    return FORGE_OK;
  });
}

int forge_sharded_scan(forge_group* g, forge_op op, int32_t inclusive, const void* const* src, void* const* dst,
                       const uint64_t* n, void* const* ws, const uint64_t* ws_bytes) {
  forge::prim::detail::NvtxRange nvtx_range("forge_sharded_scan");
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    uint32_t ss = 0;
    if (int rc = s_size_of(op, &ss); rc) return rc;
    DeviceGuard guard;
    const int G = g->size();
    if (G > 1) {
      for (int r = 0; r < G; ++r) {
        const Shard& s = g->shards[r];
        if (int rc = use(s); rc) return rc;
        if (int rc = forge_dev_reduce_ordered(op, src[r], n[r], s.local(), ws[r], ws_bytes[r], s.stream); rc)
          return rc;
      }
      if (int rc = all_gather(g, ss); rc) return rc;
      for (int r = 1; r < G; ++r) {
        const Shard& s = g->shards[r];
        if (int rc = use(s); rc) return rc;
        if (int rc = forge_dev_fold(op, s.gathered(), uint32_t(G), r, s.carry(), s.has(), s.stream); rc) return rc;
      }
    }
    for (int r = 0; r < G; ++r) {
      const Shard& s = g->shards[r];
      if (int rc = use(s); rc) return rc;
      if (int rc = forge_dev_scan(op, inclusive, src[r], dst[r], n[r], r > 0 ? s.carry() : nullptr, nullptr, ws[r],
                                  ws_bytes[r], s.stream);
          rc)
        return rc;
    }
    return FORGE_OK;
  });
}

int forge_sharded_matvec(forge_group* g, forge_op op, const void* const* A_blocks, uint64_t n, uint64_t p_cols,
                         const void* const* x, void* const* y_blocks, void* const* ws, const uint64_t* ws_bytes) {
  forge::prim::detail::NvtxRange nvtx_range("forge_sharded_matvec");
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    DeviceGuard guard;
    const int G = g->size();
    for (int r = 0; r < G; ++r) {
      uint64_t lo = 0, hi = 0;
      forge_shard_range(p_cols, r, G, &lo, &hi);
      if (hi == lo) continue;
      const Shard& s = g->shards[r];
      if (int rc = use(s); rc) return rc;
      if (int rc = forge_dev_matvec_lda(op, A_blocks[r], n, hi - lo, n, x[r], y_blocks[r], ws[r], ws_bytes[r],
                                        s.stream);
          rc)
        return rc;
    }
    return FORGE_OK;
  });
}

int forge_sharded_vecmat(forge_group* g, forge_op op, const void* const* A_blocks, uint64_t n, uint64_t p_cols,
                         const void* const* x, void* const* z_blocks, void* const* ws, const uint64_t* ws_bytes) {
  forge::prim::detail::NvtxRange nvtx_range("forge_sharded_vecmat");
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    DeviceGuard guard;
    const int G = g->size();
    for (int r = 0; r < G; ++r) {
      uint64_t lo = 0, hi = 0;
      forge_shard_range(n, r, G, &lo, &hi);
      if (hi == lo) continue;
      const Shard& s = g->shards[r];
      if (int rc = use(s); rc) return rc;
      if (int rc = forge_dev_vecmat_lda(op, A_blocks[r], hi - lo, p_cols, hi - lo, x[r], z_blocks[r], ws[r],
                                        ws_bytes[r], s.stream);
          rc)
        return rc;
    }
    return FORGE_OK;
  });
}

// ---- cross-GPU decoupled look-back over block-cyclic chunks (scan_cyclic.cuh)

int forge_cyclic_chunk_quantum(forge_op op, uint64_t* elems) {
  return guarded([&]() -> int {
    int rc = menu::visit1(op, [&](auto e) -> int {
      using T = typename decltype(e)::T;
      using S = typename decltype(e)::S;
      if constexpr (!cuda::smem_scan_type_ok<T>() || sizeof(S) != sizeof(T) || sizeof(T) > 8) {
        set_error("Unsupported: the cyclic scan takes ops with sizeof(S) == sizeof(T) <= 8");
        return FORGE_ERR_UNSUPPORTED;
      } else {
        *elems = cuda::cyclic_tile_elems<T>();
        return FORGE_OK;
      }
    });
    return rc;
  });
}

int forge_cyclic_local_n(uint64_t n, uint64_t chunk_elems, int32_t rank, int32_t count, uint64_t* local_n) {
  return guarded([&]() -> int {
    if (count <= 0 || rank < 0 || rank >= count || chunk_elems == 0 || !local_n) {
      set_error("InvalidArgument: forge_cyclic_local_n needs 0 <= rank < count and chunk_elems > 0");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    *local_n = cuda::cyclic_local_n(n, chunk_elems, uint32_t(rank), uint32_t(count));
    return FORGE_OK;
  });
}

int forge_cyclic_workspace_bytes(forge_op op, uint64_t local_n, uint64_t* bytes) {
  return guarded([&]() -> int {
    return menu::visit1(op, [&](auto e) -> int {
      using E = decltype(e);
      *bytes = cuda::cyclic_ws_bytes<typename E::T, typename E::S, typename E::Op>(local_n);
      return FORGE_OK;
    });
  });
}

int forge_sharded_scan_cyclic(forge_group* g, forge_op op, int32_t inclusive, const void* const* src,
                              void* const* dst, uint64_t n, uint64_t chunk_elems, void* const* ws,
                              const uint64_t* ws_bytes) {
  forge::prim::detail::NvtxRange nvtx_range("forge_sharded_scan_cyclic");
  return guarded([&]() -> int {
    if (int rc = check_group(g); rc) return rc;
    const int G = g->size();
    if (G > cuda::kCyclicMaxShards) {
      set_error("Unsupported: the cyclic scan takes at most 8 shards");
      return FORGE_ERR_UNSUPPORTED;
    }
    uint64_t quantum = 0;
    if (int rc = forge_cyclic_chunk_quantum(op, &quantum); rc) return rc;
    if (chunk_elems == 0 || chunk_elems % quantum) {
      set_error("InvalidArgument: chunk_elems must be a positive multiple of forge_cyclic_chunk_quantum (" +
                std::to_string(quantum) + ")");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    const uint64_t tpc = chunk_elems / quantum;
    if (tpc >= (1ull << 31) || cuda::ceil_div(n, quantum) >= (1ull << 31)) {
      set_error("InvalidArgument: too many tiles for the cyclic scan");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    if (g->emulated && tpc * uint64_t(G) > uint64_t(cuda::device_props().sm_count)) {
      // one launch deals tickets round-robin to the virtual shards: a tile may
      // wait on a ticket up to tpc * G ahead, which must be resident
      set_error("InvalidArgument: an emulated group needs chunk tiles * shards <= SM count (" +
                std::to_string(cuda::device_props().sm_count) + ")");
      return FORGE_ERR_INVALID_ARGUMENT;
    }
    DeviceGuard guard;
    if (!g->emulated && G > 1) {  // peer access: every shard reads its predecessor's tile states
      for (const Shard& a : g->shards) {
        if (int rc = use(a); rc) return rc;
        for (const Shard& b : g->shards) {
          if (a.device == b.device) continue;
          int ok = 0;
          cudaDeviceCanAccessPeer(&ok, a.device, b.device);
          if (!ok) {
            set_error("Unsupported: no peer access between the group's devices (NVLink / NVSwitch needed)");
            return FORGE_ERR_UNSUPPORTED;
          }
          const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return from_cuda(e, "peer access");
          cudaGetLastError();
        }
      }
    }
    static std::atomic<uint32_t> epochs{0};
    uint32_t epoch = 0;
    while (epoch == 0) epoch = (epochs.fetch_add(1) + 1) & 0x3fffffffu;  // process-wide, never 0
    return menu::visit1(op, [&](auto e) -> int {
      using E = decltype(e);
      using T = typename E::T;
      using S = typename E::S;
      if constexpr (!cuda::smem_scan_type_ok<T>() || sizeof(S) != sizeof(T) || sizeof(T) > 8) {
        return FORGE_ERR_UNSUPPORTED;
      } else {
        cuda::CyclicArgs<T, S, typename E::F, typename E::Op> a{};
        a.n = n;
        a.tiles = cuda::ceil_div(n, quantum);
        a.tpc = uint32_t(tpc);
        a.G = uint32_t(G);
        a.epoch = epoch;
        a.f = typename E::F{};
        a.op = typename E::Op{};
        a.identity = e.identity;
        for (int r = 0; r < G; ++r) {
          const uint64_t ln = cuda::cyclic_local_n(n, chunk_elems, uint32_t(r), uint32_t(G));
          const uint64_t need = cuda::cyclic_ws_bytes<T, S, typename E::Op>(ln);
          if (int w = require_ws(ws_bytes[r], need, "cyclic scan"); w) return w;
          a.states[r] = reinterpret_cast<uint64_t*>(static_cast<char*>(ws[r]) + 256);
          const Shard& s = g->shards[r];
          if (int rc = use(s); rc) return rc;
          if (int rc = from_cuda(cuda::ws_claim(ws[r], cuda::kWsTagScanCyclic, need, s.stream), "workspace"); rc)
            return rc;
        }
        if (g->emulated || G == 1) {
          // one launch over all (virtual) shards, on shard 0's stream
          const Shard& s0 = g->shards[0];
          if (int rc = use(s0); rc) return rc;
          std::vector<cudaEvent_t> ev(G);
          for (int r = 1; r < G; ++r) {
            cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming);
            cudaEventRecord(ev[r], g->shards[r].stream);
            cudaStreamWaitEvent(s0.stream, ev[r], 0);
          }
          a.rank0 = 0;
          a.nvirt = uint32_t(G);
          a.ctrl = static_cast<uint32_t*>(ws[0]);
          for (int r = 0; r < G; ++r) {
            a.src[r] = static_cast<const T*>(src[r]);
            a.dst[r] = static_cast<S*>(dst[r]);
            a.local_n[r] = cuda::cyclic_local_n(n, chunk_elems, uint32_t(r), uint32_t(G));
          }
          int rc = from_cuda(cuda::launch_scan_cyclic(a, inclusive != 0, s0.stream), "cyclic scan launch");
          cudaEvent_t done;
          cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
          cudaEventRecord(done, s0.stream);
          for (int r = 1; r < G; ++r) {
            cudaStreamWaitEvent(g->shards[r].stream, done, 0);
            cudaEventDestroy(ev[r]);
          }
          cudaEventDestroy(done);
          return rc;
        }
        for (int r = 0; r < G; ++r) {  // one launch per device, each over its own shard
          const Shard& s = g->shards[r];
          if (int rc = use(s); rc) return rc;
          auto ar = a;
          ar.rank0 = uint32_t(r);
          ar.nvirt = 1;
          ar.ctrl = static_cast<uint32_t*>(ws[r]);
          ar.src[0] = static_cast<const T*>(src[r]);
          ar.dst[0] = static_cast<S*>(dst[r]);
          ar.local_n[0] = cuda::cyclic_local_n(n, chunk_elems, uint32_t(r), uint32_t(G));
          if (int rc = from_cuda(cuda::launch_scan_cyclic(ar, inclusive != 0, s.stream), "cyclic scan launch"); rc)
            return rc;
        }
        return FORGE_OK;
      }
    });
  });
}

}  // extern "C"
