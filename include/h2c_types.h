/* Flat, C-ABI descriptors of the reference's H^2 data model.
 *
 * These are the plain-pointer forms of the C++ types the reference's MMP path
 * consumes and produces (proj/core/include/h2mmp/{cluster_tree,block_tree,
 * h2_matrix,mmp}.hpp).  Both the B200 library (include/h2c.h) and the CPU
 * oracle (oracle/h2o.h, test infrastructure) speak this layout, so parity
 * tests hand the very same buffers to both.
 *
 * Conventions (all follow the reference):
 *  - cluster ids are the reference's DFS pre-order ids, root = 0
 *    (cluster_tree.cpp:188-220); levels[l] lists ids ordered by `begin`;
 *  - blocks are grouped by level and sorted by (row, col) inside a level
 *    (block_tree.cpp:19-22); kind codes follow BlockKind
 *    (block_tree.hpp:13): 0 admissible, 1 inadmissible_leaf, 2 subdivided;
 *  - matrices are column-major; complex scalars are interleaved (re, im)
 *    like std::complex<double>; every offset/count is in scalars;
 *  - a leaf basis is #t x k_t, a non-leaf basis is the stacked transfer
 *    [T_c1; T_c2] of shape (k_c1 + k_c2) x k_t (h2_matrix.hpp:15-31); the root
 *    carries no basis (offset -1, rank 0);
 *  - couplings are k_t x k_s with the TRANSPOSE (not adjoint) convention on the
 *    right factor: block = V_t S V_s^T (h2_matrix.hpp:33-37).
 */
#ifndef H2C_TYPES_H
#define H2C_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { H2C_REAL = 0, H2C_COMPLEX = 1 };
enum { H2C_ADMISSIBLE = 0, H2C_INADMISSIBLE_LEAF = 1, H2C_SUBDIVIDED = 2 };

/* Return codes (mirrors the exception classes of errors.hpp:9-29 and the
 * exit-code mapping of benchmark_runner.cpp:240-254). */
enum {
  H2C_OK = 0,
  H2C_ERR_CONFIG = 2,    /* h2mmp::ConfigError    */
  H2C_ERR_INVARIANT = 3, /* h2mmp::InvariantError */
  H2C_ERR_CUDA = 4,      /* device failure (std::runtime_error on the C++ side) */
  H2C_ERR_ALLOC = 5      /* host/device allocation failure */
};

/* ClusterTree (cluster_tree.hpp:31-41). */
typedef struct h2c_tree {
  int32_t n_points;
  int32_t depth;
  int32_t leafsize;
  int32_t n_clusters;
  const int32_t* parent;   /* [n_clusters], -1 for the root */
  const int32_t* child0;   /* [n_clusters], -1 for leaves   */
  const int32_t* child1;
  const int32_t* level;
  const int32_t* begin;    /* [begin, end) in the permuted ordering */
  const int32_t* end;
  const double* bbox;      /* [n_clusters][6] = min xyz, max xyz (may be NULL) */
  const int32_t* perm;     /* [n_points] tree position -> original index */
} h2c_tree;

/* BlockTree (block_tree.hpp:40-73). */
typedef struct h2c_blocks {
  int32_t depth;
  int32_t c_sp;
  double eta;
  int64_t n_blocks;
  const int64_t* level_ptr; /* [depth + 2] */
  const int32_t* row;       /* [n_blocks] */
  const int32_t* col;
  const uint8_t* kind;
} h2c_blocks;

/* H2Matrix<Scalar> (h2_matrix.hpp:38-48).  `tree`/`blocks` are compared by
 * address, exactly like the shared_ptr identity check of mmp.cpp:59. */
typedef struct h2c_matrix {
  const h2c_tree* tree;
  const h2c_blocks* blocks;
  int32_t scalar;                /* H2C_REAL or H2C_COMPLEX */
  const int32_t* row_rank;       /* [n_clusters] */
  const int32_t* col_rank;
  const uint8_t* row_degenerate; /* [n_clusters] */
  const uint8_t* col_degenerate;
  const int64_t* row_offset;     /* [n_clusters] scalar offset into values, -1 = none */
  const int64_t* col_offset;
  const int64_t* block_offset;   /* [n_blocks] coupling or full block, -1 for subdivided */
  const double* values;
  int64_t n_values;              /* in scalars */
} h2c_matrix;

/* MmpReport + LevelStats (mmp.hpp:16-48). Per-level arrays have n_levels
 * (= depth + 1) entries; case_products is [n_levels][4]. */
typedef struct h2c_report {
  double eps_trunc;
  int32_t adaptive;
  int32_t n_levels;
  int64_t flops;            /* reference MAC counter (mmp.cpp:67-80)   */
  int64_t case_flops[4];
  double wall_seconds;
  int32_t pending_after_split;
  const int64_t* max_row_rank;
  const int64_t* max_col_rank;
  const int64_t* case_products;
  const int32_t* max_case1_terms;
  const int32_t* max_case2_terms;
  const int32_t* max_case3_terms;
  /* B200 extensions (zero in the oracle) */
  int64_t flops_exec;       /* MACs the GPU schedule actually executed */
  double device_seconds;    /* CUDA-event time of the device pipeline  */
  double plan_seconds;      /* host time spent building the structure plan (0 if cached) */
  int64_t h2d_bytes;        /* host->device bytes moved by the call */
  int64_t d2h_bytes;        /* device->host bytes moved by the call */
} h2c_report;

#ifdef __cplusplus
}
#endif

#endif /* H2C_TYPES_H */
