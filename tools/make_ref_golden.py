#!/usr/bin/env python3
"""Golden vectors from the REFERENCE ITSELF -> tests/golden/ref_cases.npz.

Runs the reference's own MMP path (/root/reference/proj/core/src, compiled
unmodified into oracle/_ref/libh2ref.so against oracle/eigen_shim; `make -C
oracle ref`) on the cases below — the instances of the reference's unit and
acceptance tests (proj/tests/test_support.hpp:37-64, test_mmp.cpp,
test_metrics.cpp:33-40, acceptance.cpp:50-64) plus the configs[0]-sized cloud
— and stores, per case: the cluster permutation and block lists, A's and C's
per-cluster ranks and degenerate flags, every MmpReport counter, the sketches
A X and C X for X = [random_vector(N, s) for s in 1..4] (metrics.cpp:17-34),
and relative_error(A, A, C, 3).  Eigenvector signs/rotations are solver
choices, so values are compared through products (sketches), never raw bases.

Run here (needs /root/reference): python tools/make_ref_golden.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from oracle import pyref as R  # noqa: E402

K = 6.283185307179586
CASES = [
    # laplace clouds (test_support.hpp laplace_cloud; tests/test_gpu_parity.py CASES)
    dict(family="random_cloud", n=256, seed=23, leafsize=25, eta=1.0, eps_h2=1e-6, eps=1e-6),
    dict(family="random_cloud", n=256, seed=1, leafsize=8, eta=1.5, eps_h2=1e-6, eps=1e-12),
    dict(family="random_cloud", n=512, seed=31, leafsize=30, eta=1.0, eps_h2=1e-6, eps=1e-4),
    dict(family="random_cloud", n=400, seed=41, leafsize=20, eta=1.0, eps_h2=1e-6, eps=1e-4),
    dict(family="random_cloud", n=128, seed=43, leafsize=16, eta=1.0, eps_h2=1e-6, eps=1e-8),
    dict(family="random_cloud", n=1024, seed=5, leafsize=16, eta=1.0, eps_h2=1e-6, eps=1e-6),
    dict(family="random_cloud", n=1024, seed=9, leafsize=12, eta=1.3, eps_h2=1e-6, eps=1e-10),
    dict(family="random_cloud", n=1024, seed=1, leafsize=30, eta=1.0, eps_h2=1e-6, eps=1e-6),
    dict(family="random_cloud", n=512, seed=31, leafsize=30, eta=1.0, eps_h2=1e-6, eps=1e-4, mode="formatted"),
    dict(family="random_cloud", n=1024, seed=9, leafsize=12, eta=1.3, eps_h2=1e-6, eps=1e-10, mode="formatted"),
    # configs[0]-sized: N = 4096 cloud, leaf 32, diagonal 0
    dict(family="random_cloud", n=4096, seed=1, leafsize=32, eta=1.0, eps_h2=1e-6, eps=1e-6, diagonal=0.0),
    # helmholtz cubes (test_support.hpp helmholtz_cube; test_mmp.cpp:61-72, :305-342)
    dict(family="cube_array", array_edge=2, cube_points=3, leafsize=20, eta=1.0, kernel="helmholtz",
         wavenumber=K, eps_h2=1e-4, eps=1e-6),
    dict(family="cube_array", array_edge=2, cube_points=3, leafsize=20, eta=1.0, kernel="helmholtz",
         wavenumber=K, eps_h2=1e-4, eps=1e-8),
    dict(family="cube_array", array_edge=2, cube_points=3, leafsize=10, eta=1.5, kernel="helmholtz",
         wavenumber=K, eps_h2=1e-6, eps=1e-12),
    dict(family="cube_array", array_edge=3, cube_points=3, leafsize=20, eta=1.0, kernel="helmholtz",
         wavenumber=K, eps_h2=1e-4, eps=1e-4),
    dict(family="cube_array", array_edge=3, cube_points=3, leafsize=20, eta=1.0, kernel="helmholtz",
         wavenumber=2.5, diagonal=3.0, eps_h2=1e-6, eps=1e-6, mode="formatted"),
    # bus and slab families (test_metrics.cpp:33-40, acceptance.cpp:66-110)
    dict(family="bus", bus_count=4, samples_per_meter=1, leafsize=30, eta=1.0, eps_h2=1e-4, eps=1e-4),
    dict(family="bus", bus_count=6, samples_per_meter=1, leafsize=30, eta=1.0, eps_h2=1e-6, eps=1e-6),
    dict(family="slab", slab_width=12, leafsize=30, eta=1.0, eps_h2=1e-4, eps=1e-6),
    dict(family="slab", slab_width=16, slab_thickness=3, leafsize=24, eta=1.2, eps_h2=1e-6, eps=1e-8),
]
GEOM_KEYS = ("family", "seed", "n", "bus_count", "samples_per_meter", "slab_width", "slab_thickness", "array_edge",
             "cube_points")


def main():
    out = {}
    meta = []
    for i, cs in enumerate(CASES):
        t0 = time.time()
        c = R.RefCase(**cs)
        cplx = c.cplx
        X = np.stack([O.random_vector(c.n, s, cplx) for s in range(1, 5)], 1)
        p = f"c{i}_"
        out[p + "perm"] = c.tree["perm"]
        for k in ("level_ptr", "row", "col", "kind"):
            out[p + "blocks_" + k] = c.blocks[k]
        ar, ac, ad, acd = c.ranks(0)
        out[p + "A_row_rank"], out[p + "A_col_rank"] = ar, ac
        out[p + "A_row_dg"], out[p + "A_col_dg"] = ad, acd
        out[p + "AX"] = c.mvp(0, X)
        cr, cc, cd, ccd = c.ranks(1)
        out[p + "C_row_rank"], out[p + "C_col_rank"] = cr, cc
        out[p + "C_row_dg"], out[p + "C_col_dg"] = cd, ccd
        out[p + "CX"] = c.mvp(1, X)
        rep = c.report()
        for k, v in rep.items():
            if k != "wall_seconds":
                out[p + "rep_" + k] = np.asarray(v)
        rel = c.relative_error(3)
        meta.append(dict(cs, c_sp=c.blocks["c_sp"], depth=c.tree["depth"], n_points=c.n,
                         relative_error_seed3=rel, ref_mmp_seconds=rep["wall_seconds"]))
        print(f"case {i}: {cs} N={c.n} flops={rep['flops']} rel={rel:.3e} ({time.time() - t0:.1f} s)", flush=True)
        del c
    assert R.shape_mismatches() == 0
    out["meta"] = np.array(json.dumps({"cases": meta, "generator": "tools/make_ref_golden.py",
                                       "reference": "proj/core/src/{geometry,cluster_tree,block_tree,h2_matrix,"
                                                    "truncation,mmp,metrics}.cpp + oracle/eigen_shim"}))
    path = os.path.join(ROOT, "tests", "golden", "ref_cases.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
