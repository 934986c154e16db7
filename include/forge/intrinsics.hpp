// forge/intrinsics.hpp — typed views, type descriptors, alignment patterns.
//
// Host half of /root/reference/proj/include/forge/intrinsics.hpp:
//   View<T>               (:19-35)   non-owning {buf, offset, length, stride}
//   TypeOf / descriptor_of (:37-66)  C++ type -> TypeDescriptor
//   make_view / create_buffer (:68-81)
//   Slot / decompose      (:114-131) 32-bit shuffle slots of a descriptor
//   LoadPattern / vload_pattern / pattern_capped (:180-211)
// The device half (shuffles, ordered loads/stores, vload_n/vstore_n) is
// replaced by direct Blackwell primitives in forge/cuda/device.cuh; when this
// header is compiled by nvcc, thin device aliases with the reference names
// (shuffle, shuffle_down, shuffle_up, ordered_load, ordered_store) are
// provided below without the VM's Ctx argument.
#pragma once

#include <array>
#include <bit>
#include <cstring>
#include <span>
#include <type_traits>
#include <vector>

#include "forge/bitstype.hpp"
#include "forge/machine.hpp"

#ifdef __CUDACC__
#include "forge/cuda/device.cuh"
#endif

namespace forge::intr {

template <class T>
struct View {
  BufferId buf = -1;
  uint64_t offset = 0;
  uint64_t length = 0;
  uint64_t stride = 1;

  bool contiguous() const { return stride == 1; }
  uint64_t index_of(uint64_t i) const { return offset + i * stride; }
  View subview(uint64_t first, uint64_t count) const {
    return View{buf, offset + first * stride, count, stride};
  }
  View strided(uint64_t first, uint64_t count, uint64_t step) const {
    return View{buf, offset + first * stride, count, stride * step};
  }
};

template <class T>
struct TypeOf;

namespace detail {
template <Scalar S>
struct ScalarTypeOf {
  static const TypeDescriptor& get() {
    static const TypeDescriptor d = TypeDescriptor::primitive(S);
    return d;
  }
};
}  // namespace detail

template <> struct TypeOf<uint8_t> : detail::ScalarTypeOf<Scalar::U8> {};
template <> struct TypeOf<int8_t> : detail::ScalarTypeOf<Scalar::U8> {};
template <> struct TypeOf<uint16_t> : detail::ScalarTypeOf<Scalar::U16> {};
template <> struct TypeOf<int16_t> : detail::ScalarTypeOf<Scalar::U16> {};
template <> struct TypeOf<uint32_t> : detail::ScalarTypeOf<Scalar::U32> {};
template <> struct TypeOf<int32_t> : detail::ScalarTypeOf<Scalar::U32> {};
template <> struct TypeOf<uint64_t> : detail::ScalarTypeOf<Scalar::U64> {};
template <> struct TypeOf<int64_t> : detail::ScalarTypeOf<Scalar::U64> {};
template <> struct TypeOf<float> : detail::ScalarTypeOf<Scalar::F32> {};
template <> struct TypeOf<double> : detail::ScalarTypeOf<Scalar::F64> {};

template <class T>
const TypeDescriptor& descriptor_of() {
  return TypeOf<T>::get();
}

template <class T>
View<T> make_view(const Machine& m, BufferId buf) {
  if (m.buffer_elem_size(buf) != sizeof(T))
    raise(ErrorCode::InvalidArgument, "view element size does not match buffer");
  return View<T>{buf, 0, m.buffer_length(buf), 1};
}

template <class T>
BufferId create_buffer(Machine& m, uint64_t length, uint32_t base_alignment = 0) {
  static_assert(std::is_trivially_copyable_v<T>, "buffers hold trivially copyable values");
  return m.create_buffer(descriptor_of<T>(), length, base_alignment);
}

// Device address of element 0 of a view (checks that the view's last element
// lies inside its buffer; the VM would fault with OutOfBounds at run time).
template <class T>
T* view_ptr(const Machine& m, const View<T>& v) {
  if (m.buffer_elem_size(v.buf) != sizeof(T))
    raise(ErrorCode::InvalidArgument, "view element size does not match buffer");
  if (v.length > 0) {
    const uint64_t last = v.offset + (v.length - 1) * v.stride;
    if (last >= m.buffer_length(v.buf)) raise(ErrorCode::InvalidArgument, "view exceeds its buffer");
  }
  return static_cast<T*>(m.device_ptr(v.buf)) + v.offset;
}

// ---------------------------------------------------------------------------
// Shuffle slots (host): every non-padding byte exactly once, 64-bit leaves as
// two slots, sub-32-bit leaves as one zero-extended slot.

struct Slot {
  uint32_t offset;
  uint32_t len;
};

std::vector<Slot> decompose(const TypeDescriptor& desc);

// ---------------------------------------------------------------------------
// Alignment patterns: greedy power-of-two segments, each
// aligned to its own size at the running element offset, capped by nitem.

struct LoadPattern {
  std::array<uint32_t, 16> seg{};
  uint32_t count = 0;
  std::span<const uint32_t> segments() const { return {seg.data(), count}; }
};

LoadPattern vload_pattern(uint64_t offset, uint32_t nitem);

namespace detail_v {

inline bool vectorizable(uint32_t esz) { return std::has_single_bit(esz); }

inline LoadPattern pattern_capped(uint64_t offset, uint32_t nitem, uint32_t max_seg) {
  LoadPattern p;
  uint64_t at = offset;
  uint32_t left = nitem;
  while (left) {
    const uint32_t align_cap =
        at == 0 ? nitem : uint32_t(std::min<uint64_t>(uint64_t(1) << std::countr_zero(at), nitem));
    const uint32_t s = std::min({align_cap, std::bit_floor(left), max_seg});
    p.seg[p.count++] = s;
    at += s;
    left -= s;
  }
  return p;
}

}  // namespace detail_v

#ifdef __CUDACC__
// Device aliases with the reference names (no Ctx: the hardware is the context).
template <class T>
__device__ __forceinline__ T shuffle(const T& value, uint32_t source_lane) {
  return cuda::shfl_idx(value, int(source_lane));
}
template <class T>
__device__ __forceinline__ T shuffle_down(const T& value, uint32_t delta) {
  return cuda::shfl_down(value, delta);
}
template <class T>
__device__ __forceinline__ T shuffle_up(const T& value, uint32_t delta) {
  return cuda::shfl_up(value, delta);
}
__device__ __forceinline__ uint32_t ordered_load(const uint32_t* p) { return cuda::ld_acquire_gpu(p); }
__device__ __forceinline__ void ordered_store(uint32_t* p, uint32_t v) { cuda::st_release_gpu(p, v); }
#endif

}  // namespace forge::intr
