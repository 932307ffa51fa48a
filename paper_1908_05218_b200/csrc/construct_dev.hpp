// Device evaluation of the interpolation couplings of the Chebyshev constructor
// (construct.cpp): S_ts = R_t K(xi_t, xi_s) R_s^T for the admissible blocks of one
// level, their row Grams sum_s S_ts S_ts^H (recompression) and the projected
// couplings P_t S_ts P_s^T.  Input side only (not the MMP path); the kernel
// matrices are evaluated by a CUDA kernel, the small dense products are batched
// cuBLAS GEMMs.
#pragma once

#include <cstdint>

namespace h2b {

struct CouplingDev;

bool cdev_available();
CouplingDev* cdev_create(bool cplx, double kappa);
void cdev_destroy(CouplingDev* d);
// clusters of one level: n clusters with boxes (center[3], half[3]) and order m
// (k = m^3 nodes); R[i] is r[i] x k column-major (host)
void cdev_level(CouplingDev* d, int n, const double* boxes, int m, const double* const* R, const int* r);
// blocks (brow[b], bcol[b]) as positions within the level, sorted by brow:
// zout[row] (r_row x r_row, interleaved complex when cplx) += sum_b S_b S_b^H
void cdev_grams(CouplingDev* d, int nb, const int* brow, const int* bcol, double* const* zout);
// P[i] is kp[i] x r[i] (column-major, interleaved complex when cplx), or nullptr for
// P = I (raw couplings); dst[b] receives P_row S_b P_col^T (kp_row x kp_col)
void cdev_project(CouplingDev* d, const double* const* P, const int* kp, int nb, const int* brow, const int* bcol,
                  double* const* dst);

}  // namespace h2b
