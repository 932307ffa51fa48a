#!/usr/bin/env python3
"""One small real and one small complex product (adaptive + formatted), an MVP and a truncation
through the C-ABI: the workload compute-sanitizer (memcheck / racecheck / synccheck) runs over
(tools/sanitize.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_05218_b200 as P

ctx = P.Context(0)
pts = P.random_cloud(2048, 1)
tree = P.build_cluster_tree(pts, 32)
st = P.build_block_tree(tree, tree, 1.0)
A = P.build_chebyshev(tree, st, pts, 3)
r = P.mmp(A, A, 1e-6, ctx)
f = P.formatted_mmp(A, A, ctx)
y = P.mvp(r.product, np.ones(2048), ctx)
Ac = P.build_chebyshev(tree, st, pts, 3, kernel="helmholtz", kappa=6.0, eps_recompress=1e-4)
rc = P.mmp(Ac, Ac, 1e-4, ctx)
b, dg = P.svd_truncate_gram(np.diag([1.0, 0.5, 1e-9, 0.0]), 1e-4, ctx)
big = np.random.default_rng(0).standard_normal((300, 120))
b2, _ = P.svd_truncate_gram(big @ big.T, 1e-8, ctx)  # cluster-distributed eigensolver path
print("sanitize workload ok", r.report.flops, rc.report.flops, b.shape, b2.shape, float(np.linalg.norm(y)))
