// bitstype.cpp — TypeDescriptor construction, layout rules and the literal
// syntax.  Contract: /root/reference/proj/include/forge/bitstype.hpp:15-71 and
// SPEC.md:159-165 (primitive <= 64 bit; tuple = natural alignment, size rounded
// to the max alignment; struct = declared offsets in order, aligned, not
// overlapping, declared size >= end of the last field).  The parser is a small
// tokenizer + recursive descent over the grammar
//   desc   := scalar | 'tuple' '(' desc (',' desc)* ')'
//           | 'struct' '(' desc '@' int (',' desc '@' int)* ';' 'size' '=' int ')'
//   scalar := u8 | u16 | u32 | u64 | f32 | f64
#include <algorithm>
#include <cctype>
#include <cstring>

#include "forge/bitstype.hpp"

namespace forge {

namespace {

struct ScalarInfo {
  Scalar s;
  const char* name;
  uint32_t bytes;
};

constexpr ScalarInfo kScalars[] = {
    {Scalar::U8, "u8", 1},   {Scalar::U16, "u16", 2}, {Scalar::U32, "u32", 4},
    {Scalar::U64, "u64", 8}, {Scalar::F32, "f32", 4}, {Scalar::F64, "f64", 8},
};

const ScalarInfo& info_of(Scalar s) {
  for (const auto& i : kScalars)
    if (i.s == s) return i;
  raise(ErrorCode::InvalidDescriptor, "unknown scalar code");
}

uint32_t round_to(uint32_t v, uint32_t a) { return a ? (v + a - 1) / a * a : v; }

void leaf_ranges(const TypeDescriptor& d, uint32_t at,
                 std::vector<std::pair<uint32_t, uint32_t>>& out) {
  if (d.kind() == TypeDescriptor::Kind::Primitive) {
    out.emplace_back(at, d.size());
    return;
  }
  for (const auto& f : d.fields()) leaf_ranges(f.type, at + f.offset, out);
}

// ---- literal parsing

enum class Tok { Word, Number, Punct, End };

struct Lexer {
  const std::string& src;
  size_t i = 0;
  Tok kind = Tok::End;
  std::string text;
  size_t at = 0;

  explicit Lexer(const std::string& s) : src(s) { next(); }

  void next() {
    while (i < src.size() && std::isspace(static_cast<unsigned char>(src[i]))) ++i;
    at = i;
    text.clear();
    if (i >= src.size()) {
      kind = Tok::End;
      return;
    }
    const char c = src[i];
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      while (i < src.size() &&
             (std::isalnum(static_cast<unsigned char>(src[i])) || src[i] == '_'))
        text += src[i++];
      kind = Tok::Word;
    } else if (std::isdigit(static_cast<unsigned char>(c))) {
      while (i < src.size() && std::isdigit(static_cast<unsigned char>(src[i]))) text += src[i++];
      kind = Tok::Number;
    } else {
      text = std::string(1, c);
      ++i;
      kind = Tok::Punct;
    }
  }

  [[noreturn]] void fail(const std::string& what) const {
    raise(ErrorCode::ParseError, "descriptor literal: " + what + " at offset " + std::to_string(at));
  }

  void punct(char c) {
    if (kind != Tok::Punct || text[0] != c) fail(std::string("expected '") + c + "'");
    next();
  }
  bool accept(char c) {
    if (kind == Tok::Punct && text[0] == c) {
      next();
      return true;
    }
    return false;
  }
  uint32_t integer() {
    if (kind != Tok::Number) fail("expected an integer");
    unsigned long long v = std::stoull(text);
    if (v > 0xffffffffull) fail("integer out of range");
    next();
    return static_cast<uint32_t>(v);
  }
  std::string word() {
    if (kind != Tok::Word) fail("expected a name");
    std::string w = text;
    next();
    return w;
  }
};

TypeDescriptor parse_desc(Lexer& lx) {
  const std::string w = lx.word();
  for (const auto& s : kScalars)
    if (w == s.name) return TypeDescriptor::primitive(s.s);
  if (w == "tuple") {
    lx.punct('(');
    std::vector<TypeDescriptor> elems;
    do elems.push_back(parse_desc(lx));
    while (lx.accept(','));
    lx.punct(')');
    return TypeDescriptor::tuple(std::move(elems));
  }
  if (w == "struct") {
    lx.punct('(');
    std::vector<TypeDescriptor::Field> fields;
    do {
      TypeDescriptor::Field f;
      f.type = parse_desc(lx);
      lx.punct('@');
      f.offset = lx.integer();
      fields.push_back(std::move(f));
    } while (lx.accept(','));
    lx.punct(';');
    if (lx.word() != "size") lx.fail("expected 'size'");
    lx.punct('=');
    const uint32_t size = lx.integer();
    lx.punct(')');
    return TypeDescriptor::struct_of(std::move(fields), size);
  }
  lx.fail("unknown type name '" + w + "'");
}

}  // namespace

uint32_t scalar_size(Scalar s) { return info_of(s).bytes; }

TypeDescriptor::TypeDescriptor() = default;

TypeDescriptor TypeDescriptor::primitive(Scalar s) {
  TypeDescriptor d;
  d.kind_ = Kind::Primitive;
  d.scalar_ = s;
  d.size_ = d.align_ = info_of(s).bytes;
  return d;
}

TypeDescriptor TypeDescriptor::tuple(std::vector<TypeDescriptor> elems) {
  if (elems.empty()) raise(ErrorCode::InvalidDescriptor, "a tuple needs at least one element");
  TypeDescriptor d;
  d.kind_ = Kind::Tuple;
  uint32_t cursor = 0, align = 1;
  d.fields_.reserve(elems.size());
  for (auto& e : elems) {
    cursor = round_to(cursor, e.alignment());
    align = std::max(align, e.alignment());
    const uint32_t sz = e.size();
    d.fields_.push_back(Field{std::move(e), cursor});
    cursor += sz;
  }
  d.align_ = align;
  d.size_ = round_to(cursor, align);
  return d;
}

TypeDescriptor TypeDescriptor::struct_of(std::vector<Field> fields, uint32_t declared_size) {
  if (fields.empty()) raise(ErrorCode::InvalidDescriptor, "a struct needs at least one field");
  uint32_t end = 0, align = 1;
  for (const auto& f : fields) {
    if (f.offset < end)
      raise(ErrorCode::InvalidDescriptor, "struct fields must be in offset order without overlap");
    if (f.offset % f.type.alignment())
      raise(ErrorCode::InvalidDescriptor, "struct field offset is not aligned for its type");
    end = f.offset + f.type.size();
    align = std::max(align, f.type.alignment());
  }
  if (declared_size < end)
    raise(ErrorCode::InvalidDescriptor, "struct size is smaller than its fields");
  TypeDescriptor d;
  d.kind_ = Kind::Struct;
  d.fields_ = std::move(fields);
  d.size_ = declared_size;
  d.align_ = align;
  return d;
}

bool TypeDescriptor::operator==(const TypeDescriptor& o) const {
  if (kind_ != o.kind_ || size_ != o.size_ || align_ != o.align_) return false;
  if (kind_ == Kind::Primitive) return scalar_ == o.scalar_;
  if (fields_.size() != o.fields_.size()) return false;
  for (size_t i = 0; i < fields_.size(); ++i)
    if (fields_[i].offset != o.fields_[i].offset || !(fields_[i].type == o.fields_[i].type))
      return false;
  return true;
}

TypeDescriptor parse_descriptor(const std::string& text) {
  Lexer lx(text);
  TypeDescriptor d = parse_desc(lx);
  if (lx.kind != Tok::End) lx.fail("unexpected trailing input");
  return d;
}

std::string to_string(const TypeDescriptor& d) {
  if (d.kind() == TypeDescriptor::Kind::Primitive) return info_of(d.scalar()).name;
  const bool is_struct = d.kind() == TypeDescriptor::Kind::Struct;
  std::string out = is_struct ? "struct(" : "tuple(";
  const auto& fs = d.fields();
  for (size_t i = 0; i < fs.size(); ++i) {
    if (i) out += ',';
    out += to_string(fs[i].type);
    if (is_struct) out += '@' + std::to_string(fs[i].offset);
  }
  if (is_struct) out += ";size=" + std::to_string(d.size());
  return out + ')';
}

std::vector<std::pair<uint32_t, uint32_t>> data_ranges(const TypeDescriptor& d) {
  std::vector<std::pair<uint32_t, uint32_t>> out;
  leaf_ranges(d, 0, out);
  return out;
}

bool value_bytes_equal(const TypeDescriptor& d, std::span<const std::byte> a,
                       std::span<const std::byte> b) {
  if (a.size() < d.size() || b.size() < d.size()) return false;
  for (const auto& [off, len] : data_ranges(d))
    if (std::memcmp(a.data() + off, b.data() + off, len) != 0) return false;
  return true;
}

}  // namespace forge
