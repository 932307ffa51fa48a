"""B200-native accuracy-controlled H^2-matrix x H^2-matrix product (arXiv 1908.05218).

Drop-in for the reference's MMP path (proj/core: h2mmp::mmp / formatted_mmp
and the H2Matrix / ClusterTree / BlockTree types).  The product runs as
level-synchronous batched sm_100a FP64 kernels behind the C-ABI of
lib/libh2mmp_b200.so; there is no CPU fallback.
"""
from .h2c import (ADMISSIBLE, INADMISSIBLE_LEAF, SUBDIVIDED, H2C_COMPLEX, H2C_REAL, BlockTree, ClusterTree,
                  ConfigError, DeviceError, H2Matrix, InvariantError, LevelStats, MmpReport, MmpResult)
from .api import (Context, PinnedArray, ResidentOperand, build_block_tree, build_chebyshev, build_cluster_tree,
                  build_fd_laplacian, count_report, h2_to_dense, default_context, formatted_mmp, mmp, mmp_resident, mvp, pin_matrix, plan_stats, random_cloud, random_vector, relative_error,
                  svd_truncate_gram, target_status)

__all__ = [
    "ADMISSIBLE", "INADMISSIBLE_LEAF", "SUBDIVIDED", "H2C_REAL", "H2C_COMPLEX", "BlockTree", "ClusterTree",
    "ConfigError", "DeviceError", "H2Matrix", "InvariantError", "LevelStats", "MmpReport", "MmpResult", "Context",
    "PinnedArray", "ResidentOperand", "build_block_tree", "build_chebyshev", "build_cluster_tree", "h2_to_dense",
    "build_fd_laplacian", "count_report", "default_context", "formatted_mmp", "mmp", "mmp_resident", "mvp", "pin_matrix", "random_vector", "relative_error", "svd_truncate_gram", "plan_stats", "random_cloud", "target_status",
]
