// Exception types of the nuspectral interface (reference: include/nuspectral/errors.hpp:9-49).
// The B200 library reports failures as C-ABI status codes (include/nus_c.h); the
// C++ layer rethrows them as exactly these types.
#pragma once

#include <stdexcept>
#include <string>

namespace nuspectral {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

class ConditioningError : public Error {
 public:
  using Error::Error;
};

class SpectralRangeError : public Error {
 public:
  using Error::Error;
};

class ExtrapolationError : public Error {
 public:
  using Error::Error;
};

class PlanMismatch : public Error {
 public:
  using Error::Error;
};

class DegenerateTapers : public Error {
 public:
  using Error::Error;
};

class BandRangeError : public Error {
 public:
  using Error::Error;
};

/// CUDA runtime / device failure (no reference counterpart: the reference never leaves the CPU).
class DeviceError : public Error {
 public:
  using Error::Error;
};

}  // namespace nuspectral
