"""Quick GPU parity probe: B200 product vs oracle on small seeded instances."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import pyoracle as O
import paper_1908_05218_b200 as P

def rel(x, y):
    return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)

cases = [(256, 23, 25, 1.0, 1e-6), (256, 1, 8, 1.5, 1e-12), (512, 31, 30, 1.0, 1e-4), (400, 41, 20, 1.0, 1e-4),
         (128, 43, 16, 1.0, 1e-8), (1024, 5, 16, 1.0, 1e-6)]
for (n, seed, leaf, eta, eps) in cases:
    pts = O.geometry("random_cloud", seed=seed, n=n)
    t = O.build_cluster_tree(pts, leaf); s = O.build_block_tree(t, eta)
    A = O.build_h2(O.assemble_dense(pts), s, 1e-6)
    da = O.h2_to_dense(A); ref = da @ da
    for adaptive in (True, False):
        ro = O.mmp(A, A, eps, adaptive=adaptive)
        t0 = time.time()
        rg = P.mmp(A, A, eps) if adaptive else P.formatted_mmp(A, A)
        dt = time.time() - t0
        co = O.h2_to_dense(ro.product); cg = O.h2_to_dense(rg.product)
        same_ranks = np.array_equal(ro.product.row_rank, rg.product.row_rank) and np.array_equal(ro.product.col_rank, rg.product.col_rank)
        print(f"n={n} leaf={leaf} eta={eta} eps={eps} adaptive={adaptive}: gpu-vs-oracle {rel(cg, co):.2e} "
              f"oracle-vs-dense {rel(co, ref):.2e} gpu-vs-dense {rel(cg, ref):.2e} ranks_equal={same_ranks} "
              f"flops_equal={rg.report.flops == ro.report.flops} t={dt*1e3:.1f}ms", flush=True)
