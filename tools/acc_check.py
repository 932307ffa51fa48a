"""Accuracy / determinism probe on a Chebyshev workload: GPU vs oracle (MVP eps_rel)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1908_05218_b200 as P
from oracle import pyoracle as O
n = int(sys.argv[1]); leaf = int(sys.argv[2]); order = int(sys.argv[3]); eps = float(sys.argv[4])
run_oracle = len(sys.argv) > 5 and sys.argv[5] == "oracle"
pts = P.random_cloud(n, 1)
t = P.build_cluster_tree(pts, leaf); s = P.build_block_tree(t, t, 1.0)
A = P.build_chebyshev(t, s, pts, order)
ctx = P.Context(0)
r1 = P.mmp(A, A, eps, ctx)
r2 = P.mmp(A, A, eps, ctx)
print("deterministic ranks:", np.array_equal(r1.product.row_rank, r2.product.row_rank),
      "values identical:", np.array_equal(r1.product.values, r2.product.values), flush=True)
def erel(C, seed=5):
    x = O.random_vector(n, seed)
    ref = O.mvp(A, O.mvp(A, x))
    return np.linalg.norm(O.mvp(C, x) - ref) / np.linalg.norm(ref)
print("gpu eps_rel", erel(r1.product), "levels", [(l.max_row_rank, l.max_col_rank) for l in r1.report.levels], flush=True)
if run_oracle:
    t0 = time.time()
    ro, margin = O.mmp(A, A, eps, with_margin=True)
    print("oracle time", time.time() - t0, "margin", margin, flush=True)
    print("oracle eps_rel", erel(ro.product), "levels", [(l.max_row_rank, l.max_col_rank) for l in ro.report.levels])
    print("ranks equal:", np.array_equal(ro.product.row_rank, r1.product.row_rank),
          "n differing clusters:", int(np.sum(ro.product.row_rank != r1.product.row_rank)))
    x = O.random_vector(n, 9)
    d = O.mvp(r1.product, x) - O.mvp(ro.product, x)
    print("gpu-vs-oracle mvp rel", np.linalg.norm(d) / np.linalg.norm(O.mvp(ro.product, x)))
# where do the two GPU runs differ?
t_ = A.tree
for l, ids in enumerate(t_.levels):
    a, b = r1.product.row_rank[ids], r2.product.row_rank[ids]
    if not np.array_equal(a, b):
        print("level", l, "rank differences at", int(np.sum(a != b)), "clusters", flush=True)
