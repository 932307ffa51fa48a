"""Pins the CPU oracle (oracle/, a restatement of the reference) against the
reference's own known-answer and property tests for the MMP path.

The reference ships no golden vectors and cannot be compiled here (Eigen is
absent), so the oracle is pinned by every KAT and bound the
reference's tests hold:
  proj/tests/test_truncation.cpp:10-66, test_trees.cpp:30-174,
  test_metrics.cpp:79-114, test_mmp.cpp:21-409, acceptance.cpp:50-201.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1908_05218_b200.h2c import ADMISSIBLE, INADMISSIBLE_LEAF, ConfigError


def laplace_cloud(n, seed, leafsize=30, eta=1.0, eps_h2=1e-4):
    """test_support.hpp:49-52"""
    pts = O.geometry("random_cloud", seed=seed, n=n)
    t = O.build_cluster_tree(pts, leafsize)
    s = O.build_block_tree(t, eta)
    d = O.assemble_dense(pts)
    return pts, t, s, d, O.build_h2(d, s, eps_h2)


def helmholtz_cube(edge, wavenumber=6.283185307179586, leafsize=20, eta=1.0, eps_h2=1e-4):
    """test_support.hpp:54-61"""
    pts = O.geometry("cube_array", array_edge=edge, cube_points=3)
    t = O.build_cluster_tree(pts, leafsize)
    s = O.build_block_tree(t, eta)
    d = O.assemble_dense(pts, "helmholtz", wavenumber)
    return pts, t, s, d, O.build_h2(d, s, eps_h2)


def rel_fro(x, ref):
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


def zero_fulls(h):
    v = h.values.copy()
    for b in range(h.structure.n_blocks):
        if h.structure.kind[b] == INADMISSIBLE_LEAF:
            o = h.block_offset[b]
            r, c = h.block(b).shape
            v[o:o + r * c] = 0
    return h.copy_with(v)


def zero_couplings(h):
    v = h.values.copy()
    for b in range(h.structure.n_blocks):
        if h.structure.kind[b] == ADMISSIBLE:
            o = h.block_offset[b]
            r, c = h.block(b).shape
            v[o:o + r * c] = 0
    return h.copy_with(v)


# ---- truncation (test_truncation.cpp) -------------------------------------
def test_truncation_known_answers():
    assert O.svd_truncate_gram(np.eye(4), 1e-2)[0].shape[1] == 4
    assert O.svd_truncate_gram(np.diag([1.0, 1e-1, 1e-3, 0.0]), 1e-2)[0].shape[1] == 2
    tie = np.diag([1.0, 1e-2])
    assert O.svd_truncate_gram(tie, 1e-2)[0].shape[1] == 1  # tie at eps is dropped
    assert O.svd_truncate_gram(tie, 0.5e-2)[0].shape[1] == 2
    b, dg = O.svd_truncate_gram(np.zeros((5, 5)), 1e-4)
    assert dg and b.shape == (5, 1) and b[0, 0] == 1.0 and np.all(b[1:] == 0)
    rng = np.random.default_rng(42)
    m = rng.uniform(-1, 1, (6, 3))
    assert O.svd_truncate_gram(m @ m.T, 1e-12)[0].shape[1] == 3
    mc = np.array([[1 + 1j, 0 + 2j], [2 - 1j, 1], [1j, 3 + 1j], [1 - 2j, 0]])
    bc, _ = O.svd_truncate_gram(mc @ mc.conj().T, 1e-12)
    assert bc.shape[1] == 2 and np.linalg.norm(bc.conj().T @ bc - np.eye(2)) < 1e-13
    for bad in (0.0, 1.0):
        with pytest.raises(ConfigError):
            O.svd_truncate_gram(np.eye(3), bad)
    with pytest.raises(ConfigError):
        O.svd_truncate_gram(np.zeros((2, 3)), 1e-2)


# ---- trees (test_trees.cpp) ------------------------------------------------
def test_tree_known_answers():
    col = np.array([[float(i), 0, 0] for i in range(8)])
    t = O.build_cluster_tree(col, 4)
    assert t.depth == 1 and t.n_clusters == 3 and t.size(t.child0[0]) == 4 and t.size(t.child1[0]) == 4
    t5 = O.build_cluster_tree(np.array([[float(i), 0, 0] for i in range(5)]), 8)
    assert t5.depth == 0 and t5.n_clusters == 1
    pts = O.geometry("random_cloud", seed=11, n=1000)
    t = O.build_cluster_tree(pts, 30)
    assert t.depth == 6  # ceil(log2(1000/30))
    assert sorted(t.perm.tolist()) == list(range(1000))
    for lv in t.levels:
        assert np.array_equal(np.sort(t.begin[lv]), t.begin[lv])
        assert t.begin[lv][0] == 0 and t.end[lv][-1] == 1000
        assert np.all(t.end[lv][:-1] == t.begin[lv][1:])
    leaves = t.levels[t.depth]
    assert all(t.size(c) <= 30 for c in leaves)


def test_bus_suite_c_sp_is_62():
    pts = O.geometry("bus", bus_count=16, samples_per_meter=1)
    assert len(pts) == 4224
    t = O.build_cluster_tree(pts, 30)
    s = O.build_block_tree(t, 1.0)
    assert s.c_sp == 62  # test_trees.cpp:163-174
    assert s.admissible_count() > 0


def test_target_status_classification():
    # test_trees.cpp:145-160: two far-apart point groups
    pts = np.concatenate([O.geometry("random_cloud", seed=3, n=64) * 0.1,
                          O.geometry("random_cloud", seed=4, n=64) * 0.1 + 5.0])
    t = O.build_cluster_tree(pts, 8)
    s = O.build_block_tree(t, 1.0)
    left, right = int(t.child0[0]), int(t.child1[0])
    assert O.target_status(s, left, right) == 1
    ll, rr = int(t.child0[left]), int(t.child1[right])
    assert O.target_status(s, ll, rr) == 3
    assert O.target_status(s, left, left) == 2


# ---- MMP properties (test_mmp.cpp) ----------------------------------------
def test_basis_products_identity_and_definition():
    _, t, s, _, A = laplace_cloud(256, 17, 25, 1.0, 1e-6)
    bp = O.basis_products(A, A)
    for c in t.levels[t.depth]:
        k = A.row_rank[c]
        assert np.abs(bp[c] - np.eye(k)).max() < 1e-13


def test_dense_oracle_laplace():
    _, t, s, _, A = laplace_cloud(256, 23, 25, 1.0, 1e-6)
    da = O.h2_to_dense(A)
    r = O.mmp(A, A, 1e-6)
    assert rel_fro(O.h2_to_dense(r.product), da @ da) <= 1e-4
    assert r.report.pending_after_split == 0


def test_dense_oracle_complex_kernel():
    _, t, s, _, A = helmholtz_cube(2)
    da = O.h2_to_dense(A)
    ref = da @ da
    assert rel_fro(O.h2_to_dense(O.mmp(A, A, 1e-6).product), ref) <= 2e-3
    assert rel_fro(O.h2_to_dense(O.mmp(A, A, 1e-8).product), ref) <= 5e-4


def test_zero_operand_gives_zero_product():
    pts = O.geometry("random_cloud", seed=3, n=128)
    t = O.build_cluster_tree(pts, 16)
    s = O.build_block_tree(t, 1.0)
    A = O.build_h2(O.assemble_dense(pts), s, 1e-6)
    Z = O.build_h2(np.zeros((128, 128)), s, 1e-6)
    r = O.mmp(Z, A, 1e-6)
    assert np.linalg.norm(O.h2_to_dense(r.product)) <= 1e-14
    leaf = t.levels[t.depth][0]
    assert r.product.row_degenerate[leaf]
    r2 = O.mmp(A, Z, 1e-6)
    assert np.linalg.norm(O.h2_to_dense(r2.product)) <= 1e-14
    assert r2.product.col_degenerate[leaf]


def test_identity_operand_reproduces():
    _, t, s, _, A = laplace_cloud(256, 29, 25, 1.0, 1e-6)
    eye = O.build_h2(np.eye(256), s, 1e-8)
    da = O.h2_to_dense(A)
    assert rel_fro(O.h2_to_dense(O.mmp(A, eye, 1e-10).product), da) <= 1e-7
    assert rel_fro(O.h2_to_dense(O.mmp(eye, A, 1e-10).product), da) <= 1e-7


def test_monotone_in_eps():
    _, t, s, _, A = laplace_cloud(512, 31, 30, 1.0, 1e-4)
    last = 1e9
    for eps in (1e-2, 1e-4, 1e-6):
        err = O.relative_error(A, A, O.mmp(A, A, eps).product, 99)
        assert err <= last * 1.1
        last = err


def test_orthonormal_and_nested_bases():
    _, t, s, _, A = laplace_cloud(300, 37, 25, 1.0, 1e-4)
    C = O.mmp(A, A, 1e-4).product
    for c in range(t.n_clusters):
        for m in (C.row_basis(c), C.col_basis(c)):
            if m.size:
                assert np.abs(m.conj().T @ m - np.eye(m.shape[1])).max() <= 1e-12


def test_case_counts_bounded_by_c_sp():
    _, t, s, _, A = laplace_cloud(400, 41, 20, 1.0, 1e-4)
    rep = O.mmp(A, A, 1e-4).report
    for lv in rep.levels:
        assert lv.max_case1_terms <= s.c_sp ** 2
        assert lv.max_case2_terms <= s.c_sp and lv.max_case3_terms <= s.c_sp


def test_single_case_isolation():
    _, t, s, _, A = laplace_cloud(128, 43, 16, 1.0, 1e-8)
    f, r = zero_couplings(A), zero_fulls(A)
    for a, b in ((f, f), (f, r), (r, f), (r, r)):
        ref = O.h2_to_dense(a) @ O.h2_to_dense(b)
        got = O.h2_to_dense(O.mmp(a, b, 1e-12).product)
        assert np.linalg.norm(got - ref) <= 1e-10 * max(1.0, np.linalg.norm(ref))


def test_formatted_case4_collapse():
    _, t, s, _, A = laplace_cloud(192, 47, 16, 1.0, 1e-8)
    r = zero_fulls(A)
    F = O.formatted_mmp(r, r).product
    bp = O.basis_products(r, r)
    idx = s.index()
    for l in range(t.depth + 1):
        for (i, k), kind in s.level_blocks(l):
            if kind != ADMISSIBLE:
                continue
            exp = np.zeros((r.row_rank[i], r.col_rank[k]))
            for j in t.levels[l]:
                if s.kind_of(i, int(j)) == ADMISSIBLE and s.kind_of(int(j), k) == ADMISSIBLE:
                    exp += r.coupling(i, int(j)) @ bp[j] @ r.coupling(int(j), k)
            assert np.linalg.norm(F.block(idx[(i, k)]) - exp) <= 1e-12 * max(1.0, np.linalg.norm(exp))


def test_formatted_not_better_than_proposed():
    _, t, s, _, A = helmholtz_cube(2)
    ef = O.relative_error(A, A, O.formatted_mmp(A, A).product, 7)
    ep = O.relative_error(A, A, O.mmp(A, A, 1e-2).product, 7)
    assert ef >= ep


def test_nonleaf_paths_exact_real_and_complex():
    pts = O.geometry("random_cloud", seed=1, n=256)
    t = O.build_cluster_tree(pts, 8)
    s = O.build_block_tree(t, 1.5)
    A = O.build_h2(O.assemble_dense(pts), s, 1e-6)
    r = O.mmp(A, A, 1e-12)
    assert sum(sum(lv.case_products) for lv in r.report.levels if lv.level < t.depth) > 0
    d = O.h2_to_dense(A)
    assert rel_fro(O.h2_to_dense(r.product), d @ d) <= 1e-12
    cp = O.geometry("cube_array", array_edge=2, cube_points=3)
    ct = O.build_cluster_tree(cp, 10)
    cs = O.build_block_tree(ct, 1.5)
    Ac = O.build_h2(O.assemble_dense(cp, "helmholtz", 6.283185307179586), cs, 1e-6)
    dc = O.h2_to_dense(Ac)
    assert rel_fro(O.h2_to_dense(O.mmp(Ac, Ac, 1e-12).product), dc @ dc) <= 1e-12


def test_asymmetric_complex_operands():
    cp = O.geometry("cube_array", array_edge=2, cube_points=3)
    t = O.build_cluster_tree(cp, 10)
    s = O.build_block_tree(t, 1.5)
    A = O.build_h2(O.assemble_dense(cp, "helmholtz", 6.283185307179586), s, 1e-6)
    B = O.build_h2(O.assemble_dense(cp, "helmholtz", 2.5, diagonal=3.0), s, 1e-6)
    ref = O.h2_to_dense(A) @ O.h2_to_dense(B)
    r = O.mmp(A, B, 1e-12)
    assert rel_fro(O.h2_to_dense(r.product), ref) <= 1e-12
    ef = O.relative_error(A, B, O.formatted_mmp(A, B).product, 3)
    assert O.relative_error(A, B, r.product, 3) <= ef


def test_operands_must_share_trees_and_eps_range():
    pts = O.geometry("random_cloud", seed=71, n=64)
    t1, t2 = O.build_cluster_tree(pts, 8), O.build_cluster_tree(pts, 8)
    s1, s2 = O.build_block_tree(t1, 1.0), O.build_block_tree(t2, 1.0)
    d = O.assemble_dense(pts)
    A, B = O.build_h2(d, s1, 1e-4), O.build_h2(d, s2, 1e-4)
    with pytest.raises(ConfigError):
        O.mmp(A, B, 1e-4)
    for bad in (0.0, 1.0):
        with pytest.raises(ConfigError):
            O.mmp(A, A, bad)


def test_case4_flop_formula():
    # test_metrics.cpp:79-114
    _, t, s, _, A = laplace_cloud(256, 13, 25, 1.0, 1e-4)
    r = O.mmp(A, A, 1e-4)
    C = r.product
    exp = 0
    for l in range(t.depth + 1):
        blocks = s.level_blocks(l)
        for j in t.levels[l]:
            for (i, jj), ka in blocks:
                if jj != j or ka != ADMISSIBLE:
                    continue
                for (j2, k), kb in blocks:
                    if j2 != j or kb != ADMISSIBLE:
                        continue
                    kc, kai, kaj = C.row_rank[i], A.row_rank[i], A.col_rank[j]
                    kbj, kbk, kck = A.row_rank[j], A.col_rank[k], C.col_rank[k]
                    exp += kc * kai * kaj + kc * kaj * kbj + kc * kbj * kbk + kc * kbk * kck
    assert r.report.case_flops[3] == exp
    assert r.report.flops > sum(r.report.case_flops)


def test_exact_rows_in_span_of_new_bases():
    _, t, s, _, A = laplace_cloud(512, 73, 30, 1.0, 1e-6)
    da = O.h2_to_dense(A)
    ref = (da @ da)[np.ix_(t.perm, t.perm)]
    C = O.mmp(A, A, 1e-12).product
    for c in t.levels[t.depth]:
        far = []
        a = int(c)
        while a >= 0:
            for (i, k), kind in s.level_blocks(int(t.level[a])):
                if kind == ADMISSIBLE and i == a:
                    far.append((t.begin[k], t.size(k)))
            a = int(t.parent[a])
        if not far:
            continue
        rows = np.concatenate([ref[t.begin[c]:t.end[c], b:b + n] for b, n in far], axis=1)
        v = C.row_basis(int(c))
        assert np.linalg.norm(rows - v @ (v.conj().T @ rows)) / np.linalg.norm(rows) <= 1e-10


def test_mvp_matches_dense():
    # acceptance.cpp:179-201 (criterion 6)
    pts, t, s, d, A = laplace_cloud(512, 5, 30, 1.0, 1e-6)
    x = O.random_vector(512, 11)
    assert np.linalg.norm(O.mvp(A, x) - O.h2_to_dense(A) @ x) <= 1e-11 * np.linalg.norm(O.h2_to_dense(A) @ x)
