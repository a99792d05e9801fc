// stengrid/errors.hpp — the reference's exception types, raised from C ABI
// statuses (include/stengrid/sg.h) so C++ callers see exactly what the
// reference throws: std::invalid_argument, std::logic_error,
// PentaSolveError{system} (penta.hpp:51-55), std::domain_error.
#pragma once

#include <stdexcept>
#include <string>

#include "stengrid/sg.h"

namespace stengrid {

struct PentaSolveError : std::runtime_error {
  int system;
  PentaSolveError(const std::string& what, int system_) : std::runtime_error(what), system(system_) {}
};

/// No CUDA device / CUDA failure: there is no CPU fallback.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
[[noreturn]] inline void throw_status(sg_status s) {
  const std::string msg = sg_last_error();
  switch (s) {
    case SG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SG_ERR_LOGIC: throw std::logic_error(msg);
    case SG_ERR_PENTA_SOLVE: throw PentaSolveError(msg, sg_last_error_system());
    case SG_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw DeviceError(msg);
  }
}
inline void check(sg_status s) {
  if (s != SG_OK) throw_status(s);
}
}  // namespace detail

}  // namespace stengrid
