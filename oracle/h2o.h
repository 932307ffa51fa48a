/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * C-ABI of the CPU oracle (a restatement of the reference's MMP path, see
 * oracle/product_engine.cpp).  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline legs load liboracle.so, and only as the checker.
 * It speaks the same flat descriptors as the B200 library (include/h2c_types.h).
 */
#ifndef H2O_H
#define H2O_H

#include "../include/h2c_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2o_tree h2o_tree;
typedef struct h2o_blocks h2o_blocks;
typedef struct h2o_matrix h2o_matrix;
typedef struct h2o_result h2o_result;

const char* h2o_last_error(void);
void h2o_set_threads(int n); /* OpenBLAS threads (reference: single-threaded) */
/* threads of the parallel restatement of the product (default 1; results are
 * bit-identical for any count, see oracle/product_engine.cpp) */
void h2o_set_mmp_threads(int n);

/* geometry.cpp:141-181; family: 0 random_cloud, 1 bus, 2 slab, 3 cube_array */
int64_t h2o_geometry_count(int family, uint64_t seed, int n, int bus_count, int samples_per_meter,
                           int slab_width, int slab_thickness, int array_edge, int cube_points);
int h2o_geometry_fill(int family, uint64_t seed, int n, int bus_count, int samples_per_meter,
                      int slab_width, int slab_thickness, int array_edge, int cube_points,
                      double* xyz);
/* geometry.cpp:200-233; kind 0 laplace (real), 1 helmholtz (complex) */
int h2o_assemble_dense(const double* xyz, int n, int kind, double wavenumber, int has_diagonal,
                       double diagonal, double* out);

/* cluster_tree.cpp:66-93 / block_tree.cpp:9-53 */
h2o_tree* h2o_build_tree(const double* xyz, int n, int leafsize);
void h2o_tree_desc(const h2o_tree* t, h2c_tree* out);
void h2o_tree_free(h2o_tree* t);
h2o_blocks* h2o_build_blocks(const h2c_tree* tree, double eta);
void h2o_blocks_desc(const h2o_blocks* b, h2c_blocks* out);
void h2o_blocks_free(h2o_blocks* b);
/* block_tree.cpp:61-85; returns 0 full_block, 1 admissible, 2 subdivided,
 * 3 inside_admissible, <0 on error */
int h2o_target_status(const h2c_tree* tree, const h2c_blocks* blocks, int t, int s);

/* h2_matrix.cpp:141-181 (small N only) */
h2o_matrix* h2o_build_h2(const h2c_tree* tree, const h2c_blocks* blocks, int scalar,
                         const double* dense, double eps_h2);
void h2o_matrix_desc(const h2o_matrix* m, h2c_matrix* out);
void h2o_matrix_free(h2o_matrix* m);

/* truncation.cpp:9-47; basis_out must hold n*n scalars */
int h2o_truncate_gram(int scalar, const double* gram, int n, double eps, double* basis_out,
                      int* rank, int* degenerate);

/* mmp.cpp:688-719.  adaptive = 1: mmp(), 0: formatted_mmp(). */
int h2o_mmp(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive,
            int64_t ff_cache_bytes, h2o_result** out);
void h2o_result_matrix(const h2o_result* r, h2c_matrix* out);
void h2o_result_report(const h2o_result* r, h2c_report* out);
double h2o_result_min_margin(const h2o_result* r);
void h2o_result_free(h2o_result* r);

/* mmp.cpp:693-714: returns total scalars; fills offsets[n_clusters],
 * rows/cols[n_clusters] and values when cap is large enough */
int64_t h2o_basis_products(const h2c_matrix* a, const h2c_matrix* b, int64_t* offsets,
                           int32_t* rows, int32_t* cols, double* values, int64_t cap);

/* h2_matrix.cpp:183-302, metrics.cpp:11-55 */
int h2o_h2_to_dense(const h2c_matrix* m, double* out);
int h2o_mvp(const h2c_matrix* m, const double* x, double* y);
int64_t h2o_memory_footprint(const h2c_matrix* m);
int h2o_random_vector(int n, uint64_t seed, int scalar, double* out);
int h2o_relative_error(const h2c_matrix* a, const h2c_matrix* b, const h2c_matrix* c,
                       uint64_t seed, double* value, int* reference_was_zero);

/* y[:, v] = A x[:, v] for nv vectors (N x nv column-major, complex interleaved) */
int h2o_mvp_multi(const h2c_matrix* m, const double* x, int nv, double* y);

/* Sliced all-cores product (bench.py CPU baseline): an engine thread runs
 * complete products C = A*B back to back with `threads` threads; each step
 * lets it run for `seconds` and returns at its next slice point with the wall
 * time, the reference MACs counted in the slice and the products completed. */
typedef struct h2o_sliced h2o_sliced;
h2o_sliced* h2o_sliced_start(const h2c_matrix* a, const h2c_matrix* b, double eps, int adaptive,
                             int threads);
int h2o_sliced_step(h2o_sliced* s, double seconds, double* elapsed, int64_t* macs,
                    int64_t* products);
void h2o_sliced_stop(h2o_sliced* s);

#ifdef __cplusplus
}
#endif

#endif
