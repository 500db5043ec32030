// parsol/errors.hpp -- error convention of the B200 solver's C++ API.
// Same codes, names and exception type as the reference
// (proj/include/parsol/errors.hpp:10-54); the C ABI returns 1 + Errc.
#pragma once

#include <stdexcept>
#include <string>

namespace parsol {

enum class Errc {
  DimensionMismatch,
  InvalidBandwidth,
  CornerForbidden,
  TooLargeForDense,
  InvalidParameter,
  ParseError,
  UnsupportedVersion,
  TooManyPartitions,
  UnsupportedKind,
  UnsupportedStructure,
  IndexOutOfRange,
  ZeroPivot,
  SingularBlock,
  SingularFactor,
  SingularReducedSystem,
  SingularWindow,
  ExhaustedBody,
  StepTooLarge,
  InvalidInterval,
  ExpmFailure,
  NotConverged,
  IoError,
  Cuda = 100,  // CUDA runtime failure (no reference equivalent)
};

const char* errc_name(Errc c);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& detail)
      : std::runtime_error(std::string(errc_name(code)) + ": " + detail), code_(code), detail_(detail) {}
  Errc code() const { return code_; }
  const std::string& detail() const { return detail_; }

 private:
  Errc code_;
  std::string detail_;
};

[[noreturn]] inline void fail(Errc code, const std::string& detail) { throw Error(code, detail); }

}  // namespace parsol
