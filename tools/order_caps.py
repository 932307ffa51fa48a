#!/usr/bin/env python3
"""configs[4] constructor with different Chebyshev order caps: per-level orders, recompressed ranks of A
and build time (decides how far the order can grow with the box size in wavelengths)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1908_05218_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
caps = [int(c) for c in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["5", "6", "7", "8"])]
pts = bench.sphere_points(n)
tree = P.build_cluster_tree(pts, 64)
st = P.build_block_tree(tree, tree, 1.0)
for hi in caps:
    orders = bench.helmholtz_orders(tree, hi=hi)
    t0 = time.perf_counter()
    A = P.build_chebyshev(tree, st, pts, orders, kernel="helmholtz", kappa=bench.KAPPA, eps_recompress=1e-4)
    dt = time.perf_counter() - t0
    mr = [int(A.row_rank[tree.level == l].max()) for l in range(1, tree.depth + 1)]
    print(json.dumps({"N": n, "cap": hi, "orders": orders.tolist(), "build_s": round(dt, 1), "max_rank_l1..": mr,
                      "values_GB": A.values.nbytes / 1e9}), flush=True)
    del A
