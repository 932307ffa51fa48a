"""The all-cores oracle (oracle/product_engine.cpp with threads > 1) is bit-identical to the
single-thread restatement of mmp.cpp (values and every MmpReport counter), its slices add up to
whole products, and bench.py's reference arm builds its inputs without the B200 library."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1908_05218_b200 as P
from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _report_equal(a, b):
    for k, v in a.__dict__.items():
        if k == "wall_seconds":
            continue
        w = b.__dict__[k]
        if isinstance(v, np.ndarray):
            assert np.array_equal(v, w), k
        else:
            assert v == w, k


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("adaptive", [True, False])
def test_parallel_oracle_bit_identical(cplx, adaptive):
    pts = P.random_cloud(2048, 3)
    tree = P.build_cluster_tree(pts, 32)
    st = P.build_block_tree(tree, tree, 1.0)
    if cplx:
        A = P.build_chebyshev(tree, st, pts, 3, kernel="helmholtz", kappa=5.0)
        B = A
    else:
        A = P.build_chebyshev(tree, st, pts, 3)
        B = P.build_chebyshev(tree, st, pts + 1e-3, 3)
    eps = 1e-5
    r1 = O.mmp(A, B, eps, adaptive=adaptive, threads=1)
    r4 = O.mmp(A, B, eps, adaptive=adaptive, threads=4)
    assert np.array_equal(r1.product.values, r4.product.values)
    assert np.array_equal(r1.product.row_rank, r4.product.row_rank)
    _report_equal(r1.report, r4.report)


def test_sliced_product_counts_whole_products():
    pts = P.random_cloud(1024, 1)
    tree = P.build_cluster_tree(pts, 32)
    st = P.build_block_tree(tree, tree, 1.0)
    A = P.build_chebyshev(tree, st, pts, 3)
    ref = O.mmp(A, A, 1e-6)
    S = O.SlicedProduct(A, A, 1e-6, 2)
    macs, prods = 0, 0
    for _ in range(200):
        el, m, prods = S.step(0.05)
        assert el > 0 and m >= 0
        macs += m
        if prods >= 2:
            break
    S.close()
    assert prods >= 2
    # the slices cover at least the completed products' counted MACs
    assert macs >= 2 * ref.report.flops


def test_reference_arm_never_maps_the_b200_library():
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import bench\n"
        "from paper_1908_05218_b200 import h2c\n"
        "h2c.use_inputs_library()\n"
        "pts, t, s, A, B = bench.build_operands('cfg5', 2048)\n"
        "from oracle import pyoracle as O\n"
        "r = O.mmp(A, B, 1e-4, threads=2)\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libh2mmp_b200' not in maps, 'B200 library mapped'\n"
        "assert 'libh2inputs' in maps and 'liboracle' in maps\n"
        "print('ok', r.report.flops)\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.startswith("ok")
