// parl/errors.hpp — drop-in for proj/include/parl/errors.hpp (errors.hpp:9-46):
// the same eight exception types, plus DeviceError for CUDA / NCCL failures
// of the device path, and the mapping from the C-ABI status codes
// (include/parl_gpu.h) back onto them.
#pragma once

#include <stdexcept>
#include <string>

#include "parl_gpu.h"

namespace parl {

#define PARL_DROPIN_ERROR(Name) \
    struct Name : std::runtime_error { explicit Name(const std::string& msg) : std::runtime_error(msg) {} };
PARL_DROPIN_ERROR(ConfigError)     // invalid or inconsistent configuration values
PARL_DROPIN_ERROR(ShapeError)      // mismatched lengths / layouts
PARL_DROPIN_ERROR(VocabError)      // token id outside the vocabulary
PARL_DROPIN_ERROR(LifecycleError)  // stale activation handle
PARL_DROPIN_ERROR(NumericError)    // NaN / Inf where a finite value is required
PARL_DROPIN_ERROR(BarrierError)    // sync / snapshot outside its barrier window
PARL_DROPIN_ERROR(StallError)      // producer / consumer watchdog
PARL_DROPIN_ERROR(IoError)         // file read / write problems
PARL_DROPIN_ERROR(DeviceError)     // CUDA / NCCL failure of the device path (no reference counterpart)
#undef PARL_DROPIN_ERROR

namespace detail {
// parl_status -> the reference exception type (message from parl_last_error)
inline void check(parl_status s, parl_ctx_t ctx = nullptr) {
    if (s == PARL_OK) return;
    const std::string m = parl_last_error(ctx);
    switch (s) {
        case PARL_E_CONFIG: throw ConfigError(m);
        case PARL_E_SHAPE: throw ShapeError(m);
        case PARL_E_VOCAB: throw VocabError(m);
        case PARL_E_LIFECYCLE: throw LifecycleError(m);
        case PARL_E_NUMERIC: throw NumericError(m);
        case PARL_E_BARRIER: throw BarrierError(m);
        case PARL_E_STALL: throw StallError(m);
        case PARL_E_IO: throw IoError(m);
        default: throw DeviceError(m);
    }
}
}  // namespace detail

}  // namespace parl
