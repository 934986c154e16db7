// forge/machine.hpp — the host boundary, backed by one CUDA device.
//
// Drop-in for the host half of /root/reference/proj/include/forge/machine.hpp:
// BufferId-addressed, zero-initialised buffers with a base alignment and an
// element descriptor (machine.hpp:151-173, machine.cpp:968-1023), and the
// LaunchReport / Fault / FaultKind / BufferCounters report types
// (machine.hpp:50-90).  The reference's VM half — the generic
// `launch(LaunchConfig, Kernel)` of host lambdas, Ctx, the Simulator and
// Threads engines, the seeded scheduler — has no B200 counterpart: real SIMT
// hardware executes the primitives' own sm_100a kernels, and there is no CPU
// fallback.  Backend / ScheduleSeed / SimTuning / TraceSink are kept as types
// so RunOptions-based call sites compile; they are accepted and ignored
// (Backend) or reinterpreted (TraceSink receives one record per kernel launch).
//
// Buffers live in HBM (cudaMalloc, over-allocated to honour base alignments
// up to 4096 B, machine.cpp:20).  write/read/fill_zero are synchronous with
// respect to the machine's stream, like the reference's host accesses.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "forge/bitstype.hpp"
#include "forge/error.hpp"

namespace forge {

enum class MemoryOrdering : uint8_t { Relaxed, Acquire, Release };
enum class Backend : uint8_t { Simulator, Threads };  // accepted, ignored on B200

const char* to_string(MemoryOrdering o);
const char* to_string(Backend b);

struct LaunchConfig {
  uint32_t num_blocks = 1;
  uint32_t threads_per_block = 32;
  uint32_t warp_width = 32;
  uint32_t shared_bytes = 0;

  uint32_t warps_per_block() const { return threads_per_block / warp_width; }
  uint64_t total_threads() const { return uint64_t(num_blocks) * threads_per_block; }
  void validate() const;
};

struct ScheduleSeed {
  uint64_t seed = 0;
  uint64_t step_budget = 100'000'000;
};

struct SimTuning {
  uint32_t max_resident_blocks = 32;
  uint32_t lane_stack_bytes = 16 * 1024;
  uint32_t drain_period = 8;
  uint32_t stale_chance = 2;
  uint32_t refetch_chance = 4;
};

enum class FaultKind : uint8_t {
  None,
  OutOfBounds,
  StepBudgetExceeded,
  BarrierDivergence,
  MisalignedVectorAccess,
  SharedMemoryExhausted,
  LaneOutOfRange,
  NonUniformWarpCall,
  Internal,  // a CUDA error (detail carries cudaGetErrorString)
};

const char* to_string(FaultKind k);

struct Fault {
  FaultKind kind = FaultKind::None;
  std::string detail;
  uint32_t block = 0;
  uint32_t thread = 0;
  int32_t buffer = -1;
  uint64_t index = 0;
};

// Per-buffer traffic.  The B200 build fills ALGORITHMIC counts for the data
// buffers a primitive touches (one load per input element, one store per
// output element); measured DRAM bytes come from ncu (profiles/).
struct BufferCounters {
  uint64_t load_events = 0;
  uint64_t load_elems = 0;
  uint64_t store_events = 0;
  uint64_t store_elems = 0;
};

struct LaunchReport {
  bool ok = false;
  Fault fault;
  uint64_t steps = 0;                   // kernel launches issued by the primitive
  std::vector<BufferCounters> buffers;  // indexed by BufferId
  double wall_seconds = 0.0;            // CUDA-event time of the primitive's kernels

  BufferCounters totals() const;
};

// One record per kernel launch: primitive name, grid, block, device seconds.
struct TraceEvent {
  uint64_t step;
  uint32_t block;  // grid size
  uint32_t warp;   // threads per block
  const char* op;  // primitive / kernel name
  int32_t buffer;
  uint64_t index;  // elements processed
  MemoryOrdering order;
  uint32_t width;
};

class TraceSink {
 public:
  virtual ~TraceSink() = default;
  virtual void on_event(const TraceEvent& e) = 0;
};

class FileTraceSink final : public TraceSink {
 public:
  explicit FileTraceSink(const std::string& path);
  ~FileTraceSink() override;
  void on_event(const TraceEvent& e) override;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

struct LaunchOptions {
  Backend backend = Backend::Simulator;
  ScheduleSeed schedule;
  SimTuning tuning;
  TraceSink* trace = nullptr;
  uint32_t thread_workers = 0;
};

using BufferId = int32_t;

class Machine {
 public:
  Machine();                    // current CUDA device
  explicit Machine(int device);
  ~Machine();
  Machine(Machine&&) noexcept;
  Machine& operator=(Machine&&) noexcept;
  Machine(const Machine&) = delete;
  Machine& operator=(const Machine&) = delete;

  BufferId create_buffer(const TypeDescriptor& elem, uint64_t length, uint32_t base_alignment = 0);
  void destroy_buffer(BufferId id);

  uint64_t buffer_length(BufferId id) const;
  uint32_t buffer_elem_size(BufferId id) const;
  uint32_t buffer_alignment(BufferId id) const;
  const TypeDescriptor& buffer_descriptor(BufferId id) const;
  size_t buffer_count() const;

  void write_bytes(BufferId id, uint64_t elem_offset, std::span<const std::byte> src);
  void read_bytes(BufferId id, uint64_t elem_offset, std::span<std::byte> dst) const;
  void fill_zero(BufferId id);

  template <class T>
  void write(BufferId id, std::span<const T> values, uint64_t elem_offset = 0) {
    write_bytes(id, elem_offset, std::as_bytes(values));
  }
  template <class T>
  void read(BufferId id, std::span<T> values, uint64_t elem_offset = 0) const {
    read_bytes(id, elem_offset, std::as_writable_bytes(values));
  }

  // ---- B200 surface used by the primitives
  void* device_ptr(BufferId id) const;  // aligned base address in HBM
  cudaStream_t stream() const;
  int device() const;
  void synchronize() const;
  // Timing: record the start / stop of a primitive's device work.
  void begin_timing();
  cudaError_t end_timing(double& seconds);  // synchronises the stream
  // Scratch device memory owned by the machine (grown on demand, reused).
  void* scratch(size_t bytes);

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

// Raised when no CUDA device is usable: the B200 layer never falls back to the CPU.
struct NoDeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Throws std::runtime_error carrying cudaGetErrorString on failure.
void check_cuda(cudaError_t e, const char* what);

}  // namespace forge
