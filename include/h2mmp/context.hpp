// The device context behind the C++ drop-in API: one h2c_context per process (the
// library's arena and call lock are per device, so every thread shares it), and the
// mapping of the C-ABI return codes to the reference's exception classes
// (errors.hpp:9-29).
#pragma once

#include <mutex>
#include <string>

#include "../h2c.h"
#include "h2mmp/errors.hpp"

namespace h2mmp {
namespace detail {

inline h2c_context* default_context() {
  struct Holder {
    h2c_context* c = nullptr;
    std::once_flag once;
    ~Holder() {
      if (c) h2c_destroy(c);
    }
  };
  static Holder h;
  std::call_once(h.once, [] {
    h.c = h2c_create(0);
    if (!h.c) throw DeviceError(h2c_last_error(nullptr));
  });
  return h.c;
}

inline void rethrow(int rc, h2c_context* ctx) {
  const std::string msg = h2c_last_error(ctx);
  switch (rc) {
    case H2C_OK: return;
    case H2C_ERR_CONFIG: throw ConfigError(msg);
    case H2C_ERR_INVARIANT: throw InvariantError(msg);
    default: throw DeviceError(msg);
  }
}

}  // namespace detail
}  // namespace h2mmp
