// machine.cu — forge::Machine on one CUDA device (see include/forge/machine.hpp).
//
// Host boundary of the reference (machine.cpp:963-1023): a table of
// zero-initialised buffers addressed by BufferId, each with a descriptor, a
// length and a base alignment (default max(4096, bit_ceil(elem)),
// machine.cpp:20, 972-973), host write/read/fill_zero with range checks
// raising InvalidArgument.  Storage is HBM; copies go through the machine's
// stream and complete before the call returns.
#include <algorithm>
#include <bit>
#include <cstdio>
#include <mutex>

#include <map>

#include "forge/cuda/device.cuh"
#include "forge/machine.hpp"

namespace forge {

namespace cuda {

cudaError_t ws_claim(void* ws, uint64_t tag, uint64_t zero_bytes, cudaStream_t stream, uint64_t extent_bytes) {
  // base address -> {layout tag, bytes zeroed for it, bytes its kernels write}
  struct Claim {
    uint64_t tag, zeroed, extent;
  };
  static std::mutex mu;
  static std::map<uintptr_t, Claim> reg;
  const uintptr_t p = reinterpret_cast<uintptr_t>(ws);
  const uint64_t extent = std::max<uint64_t>({extent_bytes, zero_bytes, 1});
  uint64_t lo = 0;  // zero [lo, zero_bytes)
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = reg.find(p);
    if (it != reg.end() && it->second.tag == tag) {
      lo = std::min(it->second.zeroed, zero_bytes);  // same layout: only bytes not zeroed before
      it->second.zeroed = std::max(it->second.zeroed, zero_bytes);
      it->second.extent = std::max(it->second.extent, extent);
    } else {
      if (it != reg.end()) reg.erase(it);
      reg[p] = Claim{tag, zero_bytes, extent};
    }
    // every other claim overlapping [p, p + extent) lost its bytes to this
    // layout: nested ones, and one below p whose extent reaches into it
    reg.erase(reg.upper_bound(p), reg.lower_bound(p + extent));
    auto at = reg.find(p);
    if (at != reg.begin()) {
      auto below = std::prev(at);
      if (below->first + below->second.extent > p) reg.erase(below);
    }
    if (reg.size() >= 4096) reg.clear();  // forgetting only costs a memset on next use
  }
  return zero_bytes > lo ? cudaMemsetAsync(static_cast<char*>(ws) + lo, 0, zero_bytes - lo, stream) : cudaSuccess;
}

}  // namespace cuda

namespace {

constexpr uint32_t kDefaultAlignment = 4096;


}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

const char* to_string(MemoryOrdering o) {
  switch (o) {
    case MemoryOrdering::Relaxed: return "rlx";
    case MemoryOrdering::Acquire: return "acq";
    case MemoryOrdering::Release: return "rel";
  }
  return "?";
}

const char* to_string(Backend b) { return b == Backend::Simulator ? "sim" : "threads"; }

const char* to_string(FaultKind k) {
  switch (k) {
    case FaultKind::None: return "none";
    case FaultKind::OutOfBounds: return "OutOfBoundsAccess";
    case FaultKind::StepBudgetExceeded: return "StepBudgetExceeded";
    case FaultKind::BarrierDivergence: return "BarrierDivergence";
    case FaultKind::MisalignedVectorAccess: return "MisalignedVectorAccess";
    case FaultKind::SharedMemoryExhausted: return "SharedMemoryExhausted";
    case FaultKind::LaneOutOfRange: return "LaneOutOfRange";
    case FaultKind::NonUniformWarpCall: return "NonUniformWarpCall";
    case FaultKind::Internal: return "InternalError";
  }
  return "?";
}

void LaunchConfig::validate() const {
  if (warp_width != 32 && warp_width != 64)
    raise(ErrorCode::InvalidArgument, "warp_width must be 32 or 64");
  if (warp_width != 32) raise(ErrorCode::Unsupported, "sm_100a warps are 32 lanes wide");
  if (num_blocks < 1) raise(ErrorCode::InvalidArgument, "num_blocks must be >= 1");
  if (threads_per_block == 0 || threads_per_block % warp_width != 0 || threads_per_block > 1024)
    raise(ErrorCode::InvalidArgument, "threads_per_block must be a multiple of 32, at most 1024");
}

BufferCounters LaunchReport::totals() const {
  BufferCounters t;
  for (const auto& c : buffers) {
    t.load_events += c.load_events;
    t.load_elems += c.load_elems;
    t.store_events += c.store_events;
    t.store_elems += c.store_elems;
  }
  return t;
}

struct FileTraceSink::Impl {
  FILE* f = nullptr;
  std::mutex mu;
};

FileTraceSink::FileTraceSink(const std::string& path) : impl_(new Impl) {
  impl_->f = std::fopen(path.c_str(), "w");
  if (!impl_->f) raise(ErrorCode::InvalidArgument, "cannot open trace file " + path);
  std::fprintf(impl_->f, "step\tgrid\tthreads\top\tbuffer\telements\tordering\n");
}
FileTraceSink::~FileTraceSink() {
  if (impl_ && impl_->f) std::fclose(impl_->f);
}
void FileTraceSink::on_event(const TraceEvent& e) {
  std::lock_guard<std::mutex> lock(impl_->mu);
  std::fprintf(impl_->f, "%llu\t%u\t%u\t%s\t%d\t%llu\t%s\n", (unsigned long long)e.step, e.block,
               e.warp, e.op, e.buffer, (unsigned long long)e.index, to_string(e.order));
}

struct BufferStore {
  TypeDescriptor desc;
  uint32_t esz = 0;
  uint64_t len = 0;
  uint32_t alignment = 0;
  void* raw = nullptr;
  void* base = nullptr;
  bool alive = false;
};

struct Machine::Impl {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  std::vector<BufferStore> buffers;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;

  BufferStore& at(BufferId id) {
    if (id < 0 || size_t(id) >= buffers.size() || !buffers[id].alive)
      raise(ErrorCode::InvalidArgument, "invalid buffer id " + std::to_string(id));
    return buffers[id];
  }
  const BufferStore& at(BufferId id) const { return const_cast<Impl*>(this)->at(id); }

  void select() const { check_cuda(cudaSetDevice(device), "cudaSetDevice"); }

  ~Impl() {
    if (device < 0) return;
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& b : buffers)
      if (b.alive && b.raw) cudaFree(b.raw);
    if (scratch) cudaFree(scratch);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    if (stream) cudaStreamDestroy(stream);
  }
};

static int current_device_or_throw() {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw NoDeviceError(std::string("forge: no CUDA device available (") + cudaGetErrorString(e) +
                   "); the B200 primitive layer has no CPU fallback");
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}

Machine::Machine() : Machine(current_device_or_throw()) {}

Machine::Machine(int device) : impl_(new Impl) {
  current_device_or_throw();
  impl_->device = device;
  impl_->select();
  check_cuda(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaEventCreate(&impl_->t0), "cudaEventCreate");
  check_cuda(cudaEventCreate(&impl_->t1), "cudaEventCreate");
}

Machine::~Machine() = default;
Machine::Machine(Machine&&) noexcept = default;
Machine& Machine::operator=(Machine&&) noexcept = default;

BufferId Machine::create_buffer(const TypeDescriptor& elem, uint64_t length,
                                uint32_t base_alignment) {
  const uint32_t esz = elem.size();
  if (esz == 0) raise(ErrorCode::InvalidDescriptor, "zero-size element");
  if (base_alignment == 0) base_alignment = std::max<uint32_t>(kDefaultAlignment, std::bit_ceil(esz));
  if (!std::has_single_bit(base_alignment) || base_alignment % elem.alignment() != 0)
    raise(ErrorCode::InvalidArgument,
          "base_alignment must be a power of two multiple of the element alignment");
  impl_->select();
  BufferStore b;
  b.desc = elem;
  b.esz = esz;
  b.len = length;
  b.alignment = base_alignment;
  b.alive = true;
  const uint64_t bytes = length * esz;
  if (bytes > 0) {
    // cudaMalloc returns >= 256-byte aligned memory; over-allocate for larger alignments.
    const uint64_t pad = base_alignment > 256 ? base_alignment : 0;
    check_cuda(cudaMalloc(&b.raw, bytes + pad), "cudaMalloc");
    const uintptr_t p = reinterpret_cast<uintptr_t>(b.raw);
    b.base = reinterpret_cast<void*>((p + base_alignment - 1) & ~uintptr_t(base_alignment - 1));
    check_cuda(cudaMemsetAsync(b.base, 0, bytes, impl_->stream), "cudaMemsetAsync");
    check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
  }
  impl_->buffers.push_back(std::move(b));
  return static_cast<BufferId>(impl_->buffers.size() - 1);
}

void Machine::destroy_buffer(BufferId id) {
  BufferStore& b = impl_->at(id);
  impl_->select();
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
  if (b.raw) cudaFree(b.raw);
  b.raw = b.base = nullptr;
  b.alive = false;
}

uint64_t Machine::buffer_length(BufferId id) const { return impl_->at(id).len; }
uint32_t Machine::buffer_elem_size(BufferId id) const { return impl_->at(id).esz; }
uint32_t Machine::buffer_alignment(BufferId id) const { return impl_->at(id).alignment; }
const TypeDescriptor& Machine::buffer_descriptor(BufferId id) const { return impl_->at(id).desc; }
size_t Machine::buffer_count() const { return impl_->buffers.size(); }
void* Machine::device_ptr(BufferId id) const { return impl_->at(id).base; }
cudaStream_t Machine::stream() const { return impl_->stream; }
int Machine::device() const { return impl_->device; }

void Machine::synchronize() const {
  impl_->select();
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
}

void Machine::write_bytes(BufferId id, uint64_t elem_offset, std::span<const std::byte> src) {
  BufferStore& b = impl_->at(id);
  if (src.size() % b.esz != 0 || elem_offset * b.esz + src.size() > b.len * b.esz)
    raise(ErrorCode::InvalidArgument, "host write out of range");
  if (src.empty()) return;
  impl_->select();
  check_cuda(cudaMemcpyAsync(static_cast<char*>(b.base) + elem_offset * b.esz, src.data(),
                             src.size(), cudaMemcpyHostToDevice, impl_->stream),
             "cudaMemcpyAsync H2D");
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
}

void Machine::read_bytes(BufferId id, uint64_t elem_offset, std::span<std::byte> dst) const {
  const BufferStore& b = impl_->at(id);
  if (dst.size() % b.esz != 0 || elem_offset * b.esz + dst.size() > b.len * b.esz)
    raise(ErrorCode::InvalidArgument, "host read out of range");
  if (dst.empty()) return;
  impl_->select();
  check_cuda(cudaMemcpyAsync(dst.data(), static_cast<const char*>(b.base) + elem_offset * b.esz,
                             dst.size(), cudaMemcpyDeviceToHost, impl_->stream),
             "cudaMemcpyAsync D2H");
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
}

void Machine::fill_zero(BufferId id) {
  BufferStore& b = impl_->at(id);
  if (b.len == 0) return;
  impl_->select();
  check_cuda(cudaMemsetAsync(b.base, 0, b.len * b.esz, impl_->stream), "cudaMemsetAsync");
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
}

void Machine::begin_timing() {
  impl_->select();
  check_cuda(cudaEventRecord(impl_->t0, impl_->stream), "cudaEventRecord");
}

cudaError_t Machine::end_timing(double& seconds) {
  seconds = 0.0;
  cudaError_t e = cudaEventRecord(impl_->t1, impl_->stream);
  if (e == cudaSuccess) e = cudaEventSynchronize(impl_->t1);
  if (e == cudaSuccess) e = cudaGetLastError();
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, impl_->t0, impl_->t1);
  seconds = double(ms) * 1e-3;
  return e;
}

void* Machine::scratch(size_t bytes) {
  if (bytes <= impl_->scratch_bytes && impl_->scratch) return impl_->scratch;
  impl_->select();
  check_cuda(cudaStreamSynchronize(impl_->stream), "cudaStreamSynchronize");
  if (impl_->scratch) cudaFree(impl_->scratch);
  impl_->scratch = nullptr;
  const size_t want = std::max<size_t>(bytes, 1 << 16);
  check_cuda(cudaMalloc(&impl_->scratch, want), "cudaMalloc scratch");
  check_cuda(cudaMemsetAsync(impl_->scratch, 0, want, impl_->stream), "cudaMemsetAsync");
  impl_->scratch_bytes = want;
  return impl_->scratch;
}

}  // namespace forge
