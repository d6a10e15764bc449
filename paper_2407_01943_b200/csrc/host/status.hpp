// Maps C-ABI status codes (include/nus_c.h) back to the reference's exception types.
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "nus_c.h"
#include "nuspectral/errors.hpp"

namespace nuspectral::host {

inline void check(int rc) {
  if (rc == NUS_OK) return;
  const std::string msg = nus_last_error();
  switch (rc) {
    case NUS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case NUS_ERR_PLAN_MISMATCH: throw PlanMismatch(msg);
    case NUS_ERR_BAND_RANGE: throw BandRangeError(msg);
    case NUS_ERR_EXTRAPOLATION: throw ExtrapolationError(msg);
    case NUS_ERR_NUMERIC: throw Error(msg);
    case NUS_ERR_DEGENERATE_TAPERS: throw DegenerateTapers(msg);
    case NUS_ERR_CONDITIONING: throw ConditioningError(msg);
    case NUS_ERR_SPECTRAL_RANGE: throw SpectralRangeError(msg);
    case NUS_ERR_OUT_OF_MEMORY: throw DeviceError("out of device memory: " + msg);
    default: throw DeviceError(msg);
  }
}

/// Device used by the drop-in classes: NUSPECTRAL_DEVICE (default 0).
inline int device() {
  const char* e = std::getenv("NUSPECTRAL_DEVICE");
  return e ? std::atoi(e) : 0;
}

}  // namespace nuspectral::host
