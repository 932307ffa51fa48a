// CPU-only stand-in for construct_dev.cu in the input generator library
// (oracle/_build/libh2inputs.so): no device, so construct.cpp takes its host path.
#include <stdexcept>

#include "construct_dev.hpp"

namespace h2b {
bool cdev_available() { return false; }
CouplingDev* cdev_create(bool, double) { throw std::runtime_error("no device in the input generator"); }
void cdev_destroy(CouplingDev*) {}
void cdev_level(CouplingDev*, int, const double*, int, const double* const*, const int*) {}
void cdev_grams(CouplingDev*, int, const int*, const int*, double* const*) {}
void cdev_project(CouplingDev*, const double* const*, const int*, int, const int*, const int*, double* const*) {}
}  // namespace h2b
