"""Parity against golden vectors produced by the REFERENCE ITSELF.

tests/golden/ref_cases.npz was written by tools/make_ref_golden.py from the
reference's own, unmodified MMP-path sources (/root/reference/proj/core/src)
compiled here against oracle/eigen_shim (Eigen is absent from this image;
`make -C oracle ref`).  The reference's own unit suite passes on that build
(`make -C oracle ref-tests && oracle/_ref/h2mmp_tests`: 65/65,
profiles/r02/ref_unit_tests.txt).

* CPU (`not gpu`): the oracle restatement reproduces the reference bit for bit
  where it must (cluster permutation, block lists, every rank, degenerate flag
  and MmpReport counter) and to rounding in values (sketches A X, C X).
* GPU: the CUDA product through the C-ABI, on the same inputs, reproduces the
  reference's ranks, degenerate flags and counters, and its C X to 10 eps.
"""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_cases.npz")
Z = np.load(GOLD)
META = json.loads(str(Z["meta"]))["cases"]
GEOM = ("seed", "n", "bus_count", "samples_per_meter", "slab_width", "slab_thickness", "array_edge", "cube_points")
REPORT_KEYS = ("case_flops", "max_row_rank", "max_col_rank", "case_products", "max_case1_terms", "max_case2_terms",
               "max_case3_terms")


def rel(x, ref):
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300)


def build_operand(m):
    """The reference's instance pipeline (test_support.hpp:37-47) on the oracle."""
    pts = O.geometry(m["family"], **{k: m[k] for k in GEOM if k in m})
    t = O.build_cluster_tree(pts, m["leafsize"])
    s = O.build_block_tree(t, m["eta"])
    kern = m.get("kernel", "laplace")
    dense = O.assemble_dense(pts, kern, m.get("wavenumber", 0.0), m.get("diagonal"))
    return O.build_h2(dense, s, m["eps_h2"])


def probes(A, cplx):
    return np.stack([O.random_vector(A.tree.n_points, s, cplx) for s in range(1, 5)], 1)


def sketch(H, X):
    return np.stack([O.mvp(H, X[:, v]) for v in range(X.shape[1])], 1)


def check_report(i, rep):
    p = f"c{i}_rep_"
    assert rep.flops == int(Z[p + "flops"])
    assert tuple(rep.case_flops) == tuple(Z[p + "case_flops"])
    assert rep.pending_after_split == int(Z[p + "pending_after_split"])
    lv = rep.levels
    assert [x.max_row_rank for x in lv] == list(Z[p + "max_row_rank"])
    assert [x.max_col_rank for x in lv] == list(Z[p + "max_col_rank"])
    assert [list(x.case_products) for x in lv] == Z[p + "case_products"].tolist()
    assert [x.max_case1_terms for x in lv] == list(Z[p + "max_case1_terms"])
    assert [x.max_case2_terms for x in lv] == list(Z[p + "max_case2_terms"])
    assert [x.max_case3_terms for x in lv] == list(Z[p + "max_case3_terms"])


def check_product(i, C, X, tol):
    p = f"c{i}_"
    assert np.array_equal(C.row_rank, Z[p + "C_row_rank"])
    assert np.array_equal(C.col_rank, Z[p + "C_col_rank"])
    assert np.array_equal(C.row_degenerate, Z[p + "C_row_dg"])
    assert np.array_equal(C.col_degenerate, Z[p + "C_col_dg"])
    err = rel(sketch(C, X), Z[p + "CX"])
    assert err <= tol, err
    return err


IDS = [f"{m['family']}-{m.get('n') or m.get('bus_count') or m.get('slab_width') or m.get('array_edge')}-"
       f"{m.get('mode', 'mmp')}-{m['eps']:g}" for m in META]


@pytest.mark.parametrize("i", range(len(META)), ids=IDS)
def test_oracle_matches_reference(i):
    m = META[i]
    p = f"c{i}_"
    A = build_operand(m)
    assert np.array_equal(A.tree.perm, Z[p + "perm"])
    s = A.structure
    assert np.array_equal(s.level_ptr, Z[p + "blocks_level_ptr"])
    assert np.array_equal(s.row, Z[p + "blocks_row"]) and np.array_equal(s.col, Z[p + "blocks_col"])
    assert np.array_equal(s.kind, Z[p + "blocks_kind"])
    assert s.c_sp == m["c_sp"]
    assert np.array_equal(A.row_rank, Z[p + "A_row_rank"]) and np.array_equal(A.col_rank, Z[p + "A_col_rank"])
    assert np.array_equal(A.row_degenerate, Z[p + "A_row_dg"])
    assert np.array_equal(A.col_degenerate, Z[p + "A_col_dg"])
    X = probes(A, A.scalar == 1)
    assert rel(sketch(A, X), Z[p + "AX"]) <= 1e-13
    formatted = m.get("mode") == "formatted"
    r = O.formatted_mmp(A, A) if formatted else O.mmp(A, A, m["eps"])
    check_report(i, r.report)
    check_product(i, r.product, X, 1e-12)
    assert abs(O.relative_error(A, A, r.product, 3) - m["relative_error_seed3"]) <= (
        1e-9 * m["relative_error_seed3"] + 1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(META)), ids=IDS)
def test_gpu_matches_reference(i):
    import paper_1908_05218_b200 as P
    m = META[i]
    A = build_operand(m)
    ctx = P.Context(0)
    formatted = m.get("mode") == "formatted"
    r = P.formatted_mmp(A, A, ctx) if formatted else P.mmp(A, A, m["eps"], ctx)
    assert r.product.tree is A.tree and r.product.structure is A.structure
    check_report(i, r.report)
    X = probes(A, A.scalar == 1)
    check_product(i, r.product, X, 10 * max(m["eps"], 1e-14))
    # the device MVP / relative_error against the reference's metric (metrics.cpp:37-55)
    e = P.relative_error(A, A, r.product, 3, ctx)
    assert abs(e - m["relative_error_seed3"]) <= 1e-6 * m["relative_error_seed3"] + 10 * max(m["eps"], 1e-13)


def test_reference_arm_counts_the_reference_flops():
    """bench.py --impl reference: the shim's MAC counter over complete products equals the
    reference's own MmpReport.flops (so time windows of a running product give its true rate)."""
    from oracle import pyref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    m = META[5]
    A = build_operand(m)
    S = R.SlicedReference(A, A, m["eps"])
    total_macs, prods = 0, 0
    try:
        for _ in range(40):
            _, macs, prods, pflops = S.step(0.25)
            total_macs += macs
            if prods >= 1:
                break
    finally:
        S.close()
    assert prods >= 1 and pflops == prods * int(Z["c5_rep_flops"])
