// forge/bitstype.hpp — element layout descriptors (host side).
//
// API of /root/reference/proj/include/forge/bitstype.hpp:15-71: Scalar codes,
// TypeDescriptor {primitive <= 64 bit, tuple with natural alignment, struct
// with explicit offsets + declared size}, the literal syntax
//   u8|u16|u32|u64|f32|f64, tuple(d,...), struct(d@off,...; size=N)
// data_ranges() and padding-blind value_bytes_equal().
//
// Differences: TypeDescriptor::Field is defined after the class (the
// reference's nested by-value member of the incomplete class does not compile
// with GCC 13), and the descriptor additionally exposes
// word_count() = ceil(size / 4), the number of 32-bit words a warp shuffle of
// the value moves on sm_100a (padding included; intrinsics.hpp:114-131 used
// per-field slots instead).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "forge/error.hpp"

namespace forge {

enum class Scalar : uint8_t { U8, U16, U32, U64, F32, F64 };

uint32_t scalar_size(Scalar s);

class TypeDescriptor {
 public:
  enum class Kind : uint8_t { Primitive, Tuple, Struct };
  struct Field;

  static TypeDescriptor primitive(Scalar s);
  static TypeDescriptor tuple(std::vector<TypeDescriptor> elems);
  static TypeDescriptor struct_of(std::vector<Field> fields, uint32_t declared_size);

  Kind kind() const { return kind_; }
  Scalar scalar() const { return scalar_; }
  uint32_t size() const { return size_; }
  uint32_t alignment() const { return align_; }
  uint32_t word_count() const { return (size_ + 3) / 4; }
  const std::vector<Field>& fields() const { return fields_; }

  bool operator==(const TypeDescriptor& other) const;

  TypeDescriptor();

 private:
  Kind kind_ = Kind::Primitive;
  Scalar scalar_ = Scalar::U32;
  uint32_t size_ = 4;
  uint32_t align_ = 4;
  std::vector<Field> fields_;
};

struct TypeDescriptor::Field {
  TypeDescriptor type;
  uint32_t offset = 0;
};

TypeDescriptor parse_descriptor(const std::string& text);
std::string to_string(const TypeDescriptor& desc);

std::vector<std::pair<uint32_t, uint32_t>> data_ranges(const TypeDescriptor& desc);

bool value_bytes_equal(const TypeDescriptor& desc, std::span<const std::byte> a,
                       std::span<const std::byte> b);

}  // namespace forge
