// Host-only entry points of include/h2c.h that build the structure and the
// synthetic BASELINE inputs (no device code).  Compiled into libh2mmp_b200.so
// and, on its own with construct_dev_stub.cpp, into the CPU-only input
// generator oracle/_build/libh2inputs.so that bench.py's reference arm uses
// (so that arm never maps the B200 library).
#pragma once

#include <memory>
#include <string>

#include "structure.hpp"

struct h2c_structure {
  std::unique_ptr<h2b::Structure> s;
};
struct h2c_h2 {
  std::unique_ptr<h2b::HostH2> m;
};

namespace h2b {
// the calling thread's last error message (h2c_last_error with a NULL context)
std::string& capi_error();
}  // namespace h2b
