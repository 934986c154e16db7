// forge/error.hpp — host-side error contract of the primitive layer.
//
// Drop-in for /root/reference/proj/include/forge/error.hpp:10-34: the same
// ErrorCode values in the same order, the same Error exception and raise().
// Device-side problems are never exceptions: they come back as
// LaunchReport{ok = false, fault} (error.hpp:8-9, machine.hpp:82-90).  Across the
// C-ABI (include/forge.h) an ErrorCode travels as status 1 + int(code).
#pragma once

#include <stdexcept>
#include <string>

namespace forge {

enum class ErrorCode {
  InvalidArgument,    // bad shape/geometry/view, non-commutative mapreduce
  InvalidDescriptor,  // malformed TypeDescriptor
  InvalidNitem,       // nitem outside {1,2,4,8,16}
  MissingIdentity,    // exclusive scan / empty reduction without identity
  WorkspaceTooSmall,  // workspace sized for a smaller problem
  DimensionMismatch,  // operand lengths disagree
  ParseError,         // descriptor literal syntax
  Unsupported,        // valid request the B200 build does not serve (warp_width 64)
};

inline const char* to_string(ErrorCode c) {
  switch (c) {
    case ErrorCode::InvalidArgument: return "InvalidArgument";
    case ErrorCode::InvalidDescriptor: return "InvalidDescriptor";
    case ErrorCode::InvalidNitem: return "InvalidNitem";
    case ErrorCode::MissingIdentity: return "MissingIdentity";
    case ErrorCode::WorkspaceTooSmall: return "WorkspaceTooSmall";
    case ErrorCode::DimensionMismatch: return "DimensionMismatch";
    case ErrorCode::ParseError: return "ParseError";
    case ErrorCode::Unsupported: return "Unsupported";
  }
  return "Unknown";
}

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const noexcept { return code_; }
  // C-ABI status (include/forge.h forge_status): 1 + code.
  int status() const noexcept { return 1 + static_cast<int>(code_); }

 private:
  ErrorCode code_;
};

[[noreturn]] inline void raise(ErrorCode code, const std::string& what) { throw Error(code, what); }

}  // namespace forge
