/* C-ABI of the B200 H^2-MMP library (libh2mmp_b200.so).
 *
 * This is the drop-in boundary for the reference's MMP path: every entry
 * point below replaces one C++ function of proj/core (cited per function);
 * plain pointers and sizes only.  Descriptors are defined in h2c_types.h.
 * The C++ API of the reference (h2mmp::mmp & co.) is restated on top of this
 * header in include/h2mmp/*.hpp; INTEGRATION.md shows the bindings.
 *
 * Every function returning int returns H2C_OK or an H2C_ERR_* code and leaves
 * a message in h2c_last_error(ctx) (thread-local when ctx is NULL).
 */
#ifndef H2C_H
#define H2C_H

#include <stddef.h>
#include <stdint.h>

#include "h2c_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2c_context h2c_context;     /* device, stream, plan cache */
typedef struct h2c_structure h2c_structure; /* owned ClusterTree + BlockTree */
typedef struct h2c_h2 h2c_h2;               /* owned H2Matrix (host, flat) */
typedef struct h2c_result h2c_result;       /* owned MmpResult (host, flat) */
typedef struct h2c_operand h2c_operand;     /* operand resident on the device */

int h2c_version(void);
const char* h2c_last_error(const h2c_context* ctx);

/* ---- context --------------------------------------------------------- */
h2c_context* h2c_create(int device);
void h2c_destroy(h2c_context* ctx);
int64_t h2c_kernel_launches(const h2c_context* ctx); /* launches of the last call */
void* h2c_stream(const h2c_context* ctx);            /* the cudaStream_t all work runs on */
/* per-launch CUDA-event profiling of the following calls (aggregated per
 * pipeline phase and kernel); entries describe the last call */
void h2c_set_profile(h2c_context* ctx, int on);
int h2c_profile_count(const h2c_context* ctx);
int h2c_profile_get(const h2c_context* ctx, int i, char* name, int cap, int64_t* launches, double* ms,
                    int64_t* macs);
/* algorithmic HBM bytes of entry i (operands read once per product entry, outputs
 * written or read+written when accumulating): the roofline's byte count */
int64_t h2c_profile_bytes(const h2c_context* ctx, int i);

/* ---- structure (host logic) ------------------------------------------
 * build_cluster_tree (cluster_tree.hpp:43, cluster_tree.cpp:66-93) followed by
 * build_block_tree(tree, tree, eta) (block_tree.hpp:75-77, block_tree.cpp:9-53).
 * xyz: [n][3] points in the original ordering.  Returns NULL on error. */
h2c_structure* h2c_build_structure(const double* xyz, int n, int leafsize, double eta);
void h2c_structure_tree(const h2c_structure* s, h2c_tree* out);
void h2c_structure_blocks(const h2c_structure* s, h2c_blocks* out);
void h2c_structure_free(h2c_structure* s);
/* BlockTree::target_status (block_tree.hpp:58, block_tree.cpp:61-85):
 * 0 full_block, 1 admissible, 2 subdivided, 3 inside_admissible, <0 error */
int h2c_target_status(const h2c_tree* tree, const h2c_blocks* blocks, int t, int s);

/* ---- synthetic inputs (not in the reference: BASELINE.json configs) ----- */
/* make_random_cloud (geometry.cpp:39-52): n points uniform in [0,1)^3 from
 * std::mt19937_64(seed), 53-bit mantissas, x,y,z per point. */
int h2c_random_cloud(int n, uint64_t seed, double* xyz);
/*
 * Nested tensor-Chebyshev H^2 matrix of order `order` (rank order^3) on the
 * cluster bounding boxes, orthonormalised bottom-up (QR; couplings
 * R_t S R_s^T) and, if eps_recompress > 0, recompressed to that accuracy.
 * kernel: 0 Laplace 1/(4 pi r), 1 Helmholtz exp(-i kappa r)/(4 pi r);
 * diagonal: value of the self term.  xyz in the original ordering. */
h2c_h2* h2c_build_chebyshev(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz,
                            int kernel, double kappa, double diagonal, int order,
                            double eps_recompress, int threads);
/* Same with an interpolation order per tree level (orders[0..depth]; e.g. growing
 * with the box size in wavelengths for Helmholtz).  With eps_recompress > 0 the
 * interpolation operand is recompressed by the rule of the reference's build_h2
 * (h2_matrix.cpp:83-121: far-field row Gram incl. inherited partners, truncated
 * by svd_truncate_gram at eps_recompress), without forming dense blocks. */
h2c_h2* h2c_build_chebyshev_orders(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz,
                                   int kernel, double kappa, double diagonal, const int* orders,
                                   double eps_recompress, int threads);
/* 7-point finite-difference Laplacian (6 on the diagonal, -1 for grid
 * neighbours) on an m x m x m grid in H^2 form: full blocks exact,
 * admissible blocks zero with rank-1 degenerate e_1 bases (the form
 * build_h2 gives an operator with no far field, h2_matrix.cpp:83-121). */
h2c_h2* h2c_build_fd_laplacian(const h2c_tree* tree, const h2c_blocks* blocks, const double* xyz,
                               double h);
void h2c_h2_desc(const h2c_h2* m, h2c_matrix* out); /* out->tree/blocks must be set by caller */
void h2c_h2_free(h2c_h2* m);

/* ---- the MMP (mmp.hpp:60-74, mmp.cpp:688-719) --------------------------
 * h2c_mmp: accuracy-controlled product C = A*B (mmp<Scalar>).  A and B must
 * share tree and blocks descriptors by ADDRESS (shared_ptr identity of
 * mmp.cpp:59) -> else H2C_ERR_CONFIG; eps must lie in (0,1).
 * h2c_formatted_mmp: baseline product with unchanged bases (formatted_mmp).
 * Host buffers in, host result out; C shares A's tree/blocks descriptors. */
int h2c_mmp(h2c_context* ctx, const h2c_matrix* a, const h2c_matrix* b, double eps_trunc,
            h2c_result** out);
int h2c_formatted_mmp(h2c_context* ctx, const h2c_matrix* a, const h2c_matrix* b,
                      h2c_result** out);
void h2c_result_matrix(const h2c_result* r, h2c_matrix* out);
void h2c_result_report(const h2c_result* r, h2c_report* out);
void h2c_result_free(h2c_result* r);

/* ---- device-resident operands (B200 extension, for repeated products) --- */
int h2c_upload(h2c_context* ctx, const h2c_matrix* m, h2c_operand** out);
void h2c_operand_free(h2c_operand* op);
/* Runs the product on resident operands; *device_seconds = CUDA-event time.
 * If out != NULL it receives the report (no matrix download). */
int h2c_mmp_resident(h2c_context* ctx, const h2c_operand* a, const h2c_operand* b,
                     double eps_trunc, int adaptive, double* device_seconds, h2c_result** out);

/* ---- svd_truncate_gram on the device (truncation.hpp:18-19, truncation.cpp:9-47) ----
 * Orthonormal eigenvectors of a Hermitian PSD Gram with lambda_i > eps*lambda_max
 * (strict, >= 1 kept, zero Gram -> e_1 + degenerate), through the same device
 * solvers the product uses.  basis_out: n x n scalars (first *rank columns set). */
int h2c_truncate_gram(h2c_context* ctx, int scalar, const double* gram, int n, double eps,
                      double* basis_out, int* rank, int* degenerate);

/* ---- exact H^2 matrix-vector product on the device (h2_matrix.cpp:213-278) ----
 * Y = A X for nv vectors; X, Y column-major N x nv in the ORIGINAL point
 * ordering (complex interleaved).  Used for the paper's eps_rel metric
 * (metrics.cpp:37-55) at sizes where a dense check is impossible. */
int h2c_mvp(h2c_context* ctx, const h2c_matrix* a, const double* x, int nv, double* y);
int h2c_mvp_resident(h2c_context* ctx, const h2c_operand* a, const double* x, int nv, double* y);
/* ---- h2_to_dense on the device (h2_matrix.cpp:124-137) -------------------
 * out = A as a dense N x N column-major matrix in the ORIGINAL point ordering
 * (complex interleaved), computed as A * I through the device MVP in column
 * panels of unit vectors generated on the device (N <= 32768). */
int h2c_to_dense(h2c_context* ctx, const h2c_matrix* a, double* out);
/* random_vector (metrics.cpp:11-35): U[-1,1] from std::mt19937_64(seed), 53-bit
 * mantissas; complex draws re then im. */
int h2c_random_vector(int n, uint64_t seed, int scalar, double* out);

/* ---- host-side accounting (no device needed) ----------------------------
 * The reference's MmpReport counters (mmp.cpp:67-80 and LevelStats) for the
 * product C = A*B, computed from the structure plan and the ranks of A, B
 * and C alone; this is what h2c_mmp reports.  Lets a CPU-only test pin the
 * plan and the counters against the oracle.  The result carries no matrix. */
int h2c_count_report(const h2c_matrix* a, const h2c_matrix* b, const h2c_matrix* c, int adaptive,
                     double eps_trunc, h2c_result** out);

/* Structure-plan statistics per level (host logic): for level l the 10
 * values out[10*l + 0..9] = clusters, admissible blocks, near blocks, pending
 * pairs, non-leaf couplings, merged pairs, R x R triples, R/F x R triples,
 * R x F triples, F x F coupling-target triples.  Returns depth+1 (levels). */
int h2c_plan_stats(const h2c_tree* tree, const h2c_blocks* blocks, int64_t* out, int cap_levels);

/* ---- pinned host memory for zero-copy-speed transfers ------------------- */
void* h2c_host_alloc(size_t bytes);
void h2c_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* H2C_H */
