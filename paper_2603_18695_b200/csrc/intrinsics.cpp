// intrinsics.cpp — host-side pieces of forge/intrinsics.hpp.
//   decompose      : SPEC.md:176-184 (slots cover every non-padding byte once;
//                    64-bit leaves -> two 32-bit slots; narrower leaves -> one
//                    zero-extended slot)
//   vload_pattern  : SPEC.md:214-222 / intrinsics.hpp:190 (nitem in {1,2,4,8,16},
//                    else InvalidNitem)
#include "forge/intrinsics.hpp"

namespace forge::intr {

namespace {

void slots_of(const TypeDescriptor& d, uint32_t at, std::vector<Slot>& out) {
  if (d.kind() != TypeDescriptor::Kind::Primitive) {
    for (const auto& f : d.fields()) slots_of(f.type, at + f.offset, out);
    return;
  }
  const uint32_t sz = d.size();
  for (uint32_t b = 0; b < sz; b += 4) out.push_back(Slot{at + b, sz - b < 4 ? sz - b : 4});
}

}  // namespace

std::vector<Slot> decompose(const TypeDescriptor& desc) {
  std::vector<Slot> out;
  slots_of(desc, 0, out);
  return out;
}

LoadPattern vload_pattern(uint64_t offset, uint32_t nitem) {
  switch (nitem) {
    case 1: case 2: case 4: case 8: case 16:
      return detail_v::pattern_capped(offset, nitem, nitem);
    default:
      raise(ErrorCode::InvalidNitem, "vload_pattern: nitem must be one of {1,2,4,8,16}");
  }
}

}  // namespace forge::intr
