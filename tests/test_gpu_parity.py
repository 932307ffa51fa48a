"""B200 parity: the CUDA product (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): identical block structure, equal per-cluster
ranks (unless an eigenvalue sits within 1e-10 of the threshold), equal
MmpReport counters, ||C_gpu - C_ref||_F / ||C_ref||_F <= 10 eps, and the dense
check against D*D at the reference's own bounds (test_mmp.cpp, acceptance.cpp).
"""
import numpy as np
import pytest

import paper_1908_05218_b200 as P
from paper_1908_05218_b200.h2c import ADMISSIBLE, INADMISSIBLE_LEAF
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return P.Context(0)


def rel(x, ref):
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300)


def structure_preserved(h):
    """test_support.hpp:133-159"""
    s, t = h.structure, h.tree
    for b in range(s.n_blocks):
        if s.kind[b] == ADMISSIBLE:
            if h.block_offset[b] < 0 or h.block(b).shape != (h.row_rank[s.row[b]], h.col_rank[s.col[b]]):
                return False
        elif s.kind[b] == INADMISSIBLE_LEAF:
            if h.block_offset[b] < 0 or h.block(b).shape != (t.size(s.row[b]), t.size(s.col[b])):
                return False
        elif h.block_offset[b] >= 0:
            return False
    return True


def check_against_oracle(A, B, eps, ctx, adaptive=True, tol=None):
    got = P.mmp(A, B, eps, ctx) if adaptive else P.formatted_mmp(A, B, ctx)
    ref, margin = O.mmp(A, B, eps, adaptive=adaptive, with_margin=True)
    C = got.product
    assert C.tree is A.tree and C.structure is A.structure  # C shares A's tree/structure (mmp.cpp:25-26)
    assert structure_preserved(C)
    if margin > 1e-10:
        assert np.array_equal(C.row_rank, ref.product.row_rank)
        assert np.array_equal(C.col_rank, ref.product.col_rank)
        assert got.report.flops == ref.report.flops
        assert got.report.case_flops == ref.report.case_flops
        for x, y in zip(got.report.levels, ref.report.levels):
            assert (x.max_row_rank, x.max_col_rank, x.case_products) == (y.max_row_rank, y.max_col_rank,
                                                                        y.case_products)
    assert np.array_equal(C.row_degenerate, ref.product.row_degenerate)
    assert np.array_equal(C.col_degenerate, ref.product.col_degenerate)
    cg, co = O.h2_to_dense(C), O.h2_to_dense(ref.product)
    err = rel(cg, co)
    assert err <= (tol if tol is not None else 10 * max(eps, 1e-14)), err
    return got, ref, cg, co


def laplace(n, seed, leaf, eta=1.0, eps_h2=1e-6):
    pts = O.geometry("random_cloud", seed=seed, n=n)
    t = O.build_cluster_tree(pts, leaf)
    s = O.build_block_tree(t, eta)
    return O.build_h2(O.assemble_dense(pts), s, eps_h2)


CASES = [(256, 23, 25, 1.0, 1e-6), (256, 1, 8, 1.5, 1e-12), (512, 31, 30, 1.0, 1e-4), (400, 41, 20, 1.0, 1e-4),
         (128, 43, 16, 1.0, 1e-8), (1024, 5, 16, 1.0, 1e-6), (1024, 9, 12, 1.3, 1e-10)]


@pytest.mark.parametrize("n,seed,leaf,eta,eps", CASES)
@pytest.mark.parametrize("adaptive", [True, False])
def test_matches_oracle(ctx, n, seed, leaf, eta, eps, adaptive):
    A = laplace(n, seed, leaf, eta)
    got, ref, cg, co = check_against_oracle(A, A, eps, ctx, adaptive)
    da = O.h2_to_dense(A)
    dense = da @ da
    assert rel(cg, dense) <= 1.1 * rel(co, dense) + 1e-13


def test_dense_oracle_bound(ctx):
    # test_mmp.cpp:50-59 / acceptance.cpp:50-64 (criterion 1)
    for n in (256, 512, 1024):
        A = laplace(n, 23, 25, 1.0, 1e-6)
        da = O.h2_to_dense(A)
        C = P.mmp(A, A, 1e-6, ctx).product
        assert rel(O.h2_to_dense(C), da @ da) <= 1e-4


def helmholtz(edge, leaf, eta, k=6.283185307179586, diag=None):
    cp = O.geometry("cube_array", array_edge=edge, cube_points=3)
    t = O.build_cluster_tree(cp, leaf)
    s = O.build_block_tree(t, eta)
    return cp, s, O.build_h2(O.assemble_dense(cp, "helmholtz", k, diag), s, 1e-6 if eta > 1 else 1e-4)


def test_complex_kernel_bounds(ctx):
    _, s, A = helmholtz(2, 20, 1.0)
    da = O.h2_to_dense(A)
    ref = da @ da
    _, _, c6, _ = check_against_oracle(A, A, 1e-6, ctx)
    assert rel(c6, ref) <= 2e-3
    _, _, c8, _ = check_against_oracle(A, A, 1e-8, ctx)
    assert rel(c8, ref) <= 5e-4


def test_nonleaf_paths_exact(ctx):
    A = laplace(256, 1, 8, 1.5)
    d = O.h2_to_dense(A)
    r = P.mmp(A, A, 1e-12, ctx)
    assert sum(sum(lv.case_products) for lv in r.report.levels if lv.level < A.tree.depth) > 0
    assert rel(O.h2_to_dense(r.product), d @ d) <= 1e-12
    cp, s, Ac = helmholtz(2, 10, 1.5)
    dc = O.h2_to_dense(Ac)
    assert rel(O.h2_to_dense(P.mmp(Ac, Ac, 1e-12, ctx).product), dc @ dc) <= 1e-12


def test_asymmetric_complex(ctx):
    cp = O.geometry("cube_array", array_edge=2, cube_points=3)
    t = O.build_cluster_tree(cp, 10)
    s = O.build_block_tree(t, 1.5)
    A = O.build_h2(O.assemble_dense(cp, "helmholtz", 6.283185307179586), s, 1e-6)
    B = O.build_h2(O.assemble_dense(cp, "helmholtz", 2.5, diagonal=3.0), s, 1e-6)
    got, _, cg, _ = check_against_oracle(A, B, 1e-12, ctx)
    assert rel(cg, O.h2_to_dense(A) @ O.h2_to_dense(B)) <= 1e-12
    C = got.product
    for c in range(t.n_clusters):
        for m in (C.row_basis(c), C.col_basis(c)):
            if m.size:
                assert np.abs(m.conj().T @ m - np.eye(m.shape[1])).max() <= 1e-12
    ef = O.relative_error(A, B, P.formatted_mmp(A, B, ctx).product, 3)
    assert O.relative_error(A, B, C, 3) <= ef


def _zero(h, kind):
    v = h.values.copy()
    for b in range(h.structure.n_blocks):
        if h.structure.kind[b] == kind:
            o = h.block_offset[b]
            r, c = h.block(b).shape
            v[o:o + r * c] = 0
    return h.copy_with(v)


def test_single_case_isolation(ctx):
    A = laplace(128, 43, 16, 1.0, 1e-8)
    f, r = _zero(A, ADMISSIBLE), _zero(A, INADMISSIBLE_LEAF)
    for a, b in ((f, f), (f, r), (r, f), (r, r)):
        ref = O.h2_to_dense(a) @ O.h2_to_dense(b)
        got = O.h2_to_dense(P.mmp(a, b, 1e-12, ctx).product)
        assert np.linalg.norm(got - ref) <= 1e-10 * max(1.0, np.linalg.norm(ref))


def test_zero_and_identity_operands(ctx):
    pts = O.geometry("random_cloud", seed=3, n=128)
    t = O.build_cluster_tree(pts, 16)
    s = O.build_block_tree(t, 1.0)
    A = O.build_h2(O.assemble_dense(pts), s, 1e-6)
    Z = O.build_h2(np.zeros((128, 128)), s, 1e-6)
    r = P.mmp(Z, A, 1e-6, ctx)
    leaf = t.levels[t.depth][0]
    assert np.linalg.norm(O.h2_to_dense(r.product)) <= 1e-14 and r.product.row_degenerate[leaf]
    r2 = P.mmp(A, Z, 1e-6, ctx)
    assert np.linalg.norm(O.h2_to_dense(r2.product)) <= 1e-14 and r2.product.col_degenerate[leaf]
    B = laplace(256, 29, 25, 1.0, 1e-6)
    eye = O.build_h2(np.eye(256), B.structure, 1e-8)
    db = O.h2_to_dense(B)
    assert rel(O.h2_to_dense(P.mmp(B, eye, 1e-10, ctx).product), db) <= 1e-7
    assert rel(O.h2_to_dense(P.mmp(eye, B, 1e-10, ctx).product), db) <= 1e-7


def test_formatted_collapse_and_dominance(ctx):
    A = laplace(192, 47, 16, 1.0, 1e-8)
    r = _zero(A, INADMISSIBLE_LEAF)
    ref = O.h2_to_dense(r) @ O.h2_to_dense(r)
    for res in (P.formatted_mmp(r, r, ctx), P.mmp(r, r, 1e-12, ctx)):
        assert np.linalg.norm(O.h2_to_dense(res.product) - ref) <= 1e-10 * max(1.0, np.linalg.norm(ref))
    _, _, H = helmholtz(2, 20, 1.0)
    assert O.relative_error(H, H, P.formatted_mmp(H, H, ctx).product, 7) >= \
        O.relative_error(H, H, P.mmp(H, H, 1e-2, ctx).product, 7)


def test_config_errors(ctx):
    pts = O.geometry("random_cloud", seed=71, n=64)
    t1, t2 = O.build_cluster_tree(pts, 8), O.build_cluster_tree(pts, 8)
    s1, s2 = O.build_block_tree(t1, 1.0), O.build_block_tree(t2, 1.0)
    d = O.assemble_dense(pts)
    A, B = O.build_h2(d, s1, 1e-4), O.build_h2(d, s2, 1e-4)
    with pytest.raises(P.ConfigError):
        P.mmp(A, B, 1e-4, ctx)
    for bad in (0.0, 1.0, -1.0):
        with pytest.raises(P.ConfigError):
            P.mmp(A, A, bad, ctx)


def test_exact_rows_in_span(ctx):
    A = laplace(512, 73, 30, 1.0, 1e-6)
    t, s = A.tree, A.structure
    da = O.h2_to_dense(A)
    ref = (da @ da)[np.ix_(t.perm, t.perm)]
    C = P.mmp(A, A, 1e-12, ctx).product
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


def chebyshev(n, leaf, order, seed=1):
    pts = P.random_cloud(n, seed)
    t = P.build_cluster_tree(pts, leaf)
    s = P.build_block_tree(t, t, 1.0)
    return P.build_chebyshev(t, s, pts, order)


def test_cfg1_parity_and_dense_check(ctx):
    """BASELINE configs[0]: N=4096, leaf 32, Chebyshev order 3 (k=27), eps=1e-6, dense check."""
    A = chebyshev(4096, 32, 3)
    got, ref, cg, co = check_against_oracle(A, A, 1e-6, ctx)
    da = O.h2_to_dense(A)
    dense = da @ da
    e_gpu, e_ref = rel(cg, dense), rel(co, dense)
    assert e_gpu <= 1.1 * e_ref + 1e-14 and e_gpu <= 1e-4, (e_gpu, e_ref)


def test_resident_path_matches_dropin(ctx):
    A = chebyshev(2048, 32, 3)
    r1 = P.mmp(A, A, 1e-6, ctx)
    dA = P.ResidentOperand(A, ctx)
    secs, rep = P.mmp_resident(dA, dA, 1e-6, want_report=True)
    assert secs > 0 and rep.flops == r1.report.flops and rep.flops_exec == r1.report.flops_exec
    assert ctx.kernel_launches() > 0


def test_cfg2_construction_at_16k_matches_oracle(ctx):
    """configs[1] construction (leaf 64, order 4 = k 64, eps 1e-8) at N=16384: full oracle parity."""
    A = chebyshev(16384, 64, 4)
    got = P.mmp(A, A, 1e-8, ctx)
    ref, margin = O.mmp(A, A, 1e-8, with_margin=True)
    C = got.product
    assert C.tree is A.tree and structure_preserved(C)
    if margin > 1e-10:
        assert np.array_equal(C.row_rank, ref.product.row_rank)
        assert np.array_equal(C.col_rank, ref.product.col_rank)
        assert got.report.flops == ref.report.flops and got.report.case_flops == ref.report.case_flops
    x = O.random_vector(16384, 9)
    yo = O.mvp(ref.product, x)
    assert np.linalg.norm(O.mvp(C, x) - yo) / np.linalg.norm(yo) <= 1e-7  # 10 eps
    ref_ax = O.mvp(A, O.mvp(A, x))
    e_gpu = np.linalg.norm(O.mvp(C, x) - ref_ax) / np.linalg.norm(ref_ax)
    e_ora = np.linalg.norm(yo - ref_ax) / np.linalg.norm(ref_ax)
    assert e_gpu <= 1.1 * e_ora + 1e-14


def test_deterministic_products(ctx):
    """Fixed-order segmented accumulation: repeated products are bit-identical."""
    A = chebyshev(8192, 64, 4)
    r1, r2 = P.mmp(A, A, 1e-8, ctx), P.mmp(A, A, 1e-8, ctx)
    assert np.array_equal(r1.product.row_rank, r2.product.row_rank)
    assert np.array_equal(r1.product.values, r2.product.values)


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_device_constructor_matches_host(name, monkeypatch):
    """The Chebyshev constructor's coupling passes on the device (kernel evaluation + batched
    GEMMs, construct_dev.cu) give the host constructor's operand: equal ranks, dense difference
    at round-off."""
    import bench
    _, _, _, Ad, Bd = bench.build_operands(name, 4096)
    monkeypatch.setenv("H2B_CONSTRUCT_HOST", "1")
    _, _, _, Ah, Bh = bench.build_operands(name, 4096)
    for d, h in ((Ad, Ah), (Bd, Bh)):
        assert np.array_equal(d.row_rank, h.row_rank) and np.array_equal(d.col_rank, h.col_rank)
        dd, dh = O.h2_to_dense(d), O.h2_to_dense(h)
        assert rel(dd, dh) <= 1e-11, rel(dd, dh)


@pytest.mark.parametrize("knob", ["H2B_CPLX4M", "H2B_NO_STRIPS_SMALL", "H2B_STRIPS_24"])
@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_small_tile_kernels_match_oracle(ctx, name, knob, monkeypatch):
    """The A/B variants (4-product complex DMMA, strip splits) on the small-rank bench constructions: oracle parity, bit-identical repeats and
    the same ranks as the default path."""
    import bench
    _, _, _, A, B = bench.build_operands(name, 4096)
    eps = bench.CONFIGS[name][3]
    monkeypatch.setenv(knob, "1")
    got, ref, cg, co = check_against_oracle(A, B, eps, ctx)
    again = P.mmp(A, B, eps, ctx)
    assert np.array_equal(again.product.values, got.product.values)
    monkeypatch.delenv(knob)
    base = P.mmp(A, B, eps, ctx)
    assert np.array_equal(base.product.row_rank, got.product.row_rank)
    assert rel(O.h2_to_dense(base.product), cg) <= 1e-12


@pytest.mark.parametrize("kind", ["real", "complex"])
def test_staged_transfers_are_exact(ctx, kind, monkeypatch):
    """Host<->device staging in bounded batches (upload sorted by source offset, download in
    destination order incl. the interleaved halves of stacked transfers) gives the same bits as
    the default 1 GiB batches."""
    if kind == "real":
        A = chebyshev(4096, 32, 3)
        eps = 1e-6
    else:
        import bench
        _, _, _, A, _ = bench.build_operands("cfg5", 4096)
        eps = 1e-4
    ref = P.mmp(A, A, eps, ctx)
    monkeypatch.setenv("H2B_STAGE_SCALARS", "3000")
    got = P.mmp(A, A, eps, ctx)
    assert np.array_equal(got.product.row_rank, ref.product.row_rank)
    assert np.array_equal(got.product.values, ref.product.values)
    monkeypatch.delenv("H2B_STAGE_SCALARS")


@pytest.mark.slow
def test_cfg2_full_size_properties(ctx):
    """configs[1] at N=65536: size-independent properties (MVP probe, orthonormality, counters, symmetry).

    The accuracy bar is relative to the oracle's own: at N=16,384 of the same construction the oracle and
    the GPU both give eps_rel = 7.7e-6 (test above); the product's truncation error does not grow with N
    beyond a small factor, so eps_rel <= 1e-4 here.
    """
    A = chebyshev(65536, 64, 4)
    r = P.mmp(A, A, 1e-8, ctx)
    C = r.product
    assert structure_preserved(C)
    assert r.report.flops == P.count_report(A, A, C, True, 1e-8).flops
    # A is symmetric (shared row/col bases) so C = A*A has equal row and column ranks
    assert np.array_equal(C.row_rank, C.col_rank)
    rng = np.random.default_rng(0)
    for c in rng.choice(np.nonzero(A.tree.parent >= 0)[0], 64, replace=False):
        for m in (C.row_basis(int(c)), C.col_basis(int(c))):
            assert np.abs(m.T @ m - np.eye(m.shape[1])).max() <= 1e-12
    for seed in (5, 6):
        x = O.random_vector(65536, seed)
        ref = O.mvp(A, O.mvp(A, x))
        assert np.linalg.norm(O.mvp(C, x) - ref) / np.linalg.norm(ref) <= 1e-4


# ---- the other BASELINE configurations at oracle-checkable sizes ------------------
def test_cfg4_like_fd_times_laplace(ctx):
    """configs[3] shape at 16^3: FD Laplacian (rank-1 degenerate far field) x Laplace H^2 (order 4)."""
    m = 16
    h = 1.0 / (m + 1)
    g = np.stack(np.meshgrid(*[np.arange(1, m + 1) * h] * 3, indexing="ij"), -1).reshape(-1, 3)
    t = P.build_cluster_tree(g, 64)
    s = P.build_block_tree(t, t, 1.0)
    A = P.build_fd_laplacian(t, s, g, h)
    B = P.build_chebyshev(t, s, g, 4)
    got, ref, cg, co = check_against_oracle(A, B, 1e-6, ctx)
    dense = O.h2_to_dense(A) @ O.h2_to_dense(B)
    assert rel(cg, dense) <= 1.1 * rel(co, dense) + 1e-13


def test_cfg3_like_plates_times_jittered(ctx):
    """configs[2] shape, small: parallel plates with centroid panels, A x B with B on jittered
    centroids built over A's tree/structure (self term 2 ln(1+sqrt2)/(pi h))."""
    nplates, m = 4, 24
    hh = 1.0 / m
    pts = []
    for p_ in range(nplates):
        for i in range(m):
            for j in range(m):
                pts.append(((i + 0.5) * hh, (j + 0.5) * hh, 0.1 * p_))
    pts = np.array(pts)
    t = P.build_cluster_tree(pts, 32)
    s = P.build_block_tree(t, t, 1.0)
    diag = 2.0 * np.log(1.0 + np.sqrt(2.0)) / (np.pi * hh)
    A = P.build_chebyshev(t, s, pts, 3, diagonal=diag)
    rng = np.random.default_rng(2)
    jit = pts + 0.05 * hh * rng.uniform(-1, 1, pts.shape)
    B = P.build_chebyshev(t, s, jit, 3, diagonal=diag)
    got, ref, cg, co = check_against_oracle(A, B, 1e-6, ctx)
    dense = O.h2_to_dense(A) @ O.h2_to_dense(B)
    assert rel(cg, dense) <= 1.1 * rel(co, dense) + 1e-13


def test_cfg5_like_helmholtz_chebyshev(ctx):
    """configs[4] shape, small: complex128 Helmholtz exp(-i k r)/(4 pi r) on a Fibonacci sphere."""
    n = 2048
    i = np.arange(n) + 0.5
    phi = np.arccos(1 - 2 * i / n)
    theta = np.pi * (1 + 5 ** 0.5) * i
    sph = 2.0 * np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi), np.cos(phi)], 1)
    t = P.build_cluster_tree(sph, 64)
    s = P.build_block_tree(t, t, 1.0)
    A = P.build_chebyshev(t, s, sph, 4, kernel="helmholtz", kappa=2 * np.pi)
    assert A.scalar == P.H2C_COMPLEX
    got, ref, cg, co = check_against_oracle(A, A, 1e-4, ctx)
    da = O.h2_to_dense(A)
    dense = da @ da
    assert rel(cg, dense) <= 1.1 * rel(co, dense) + 1e-13


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_bench_constructions_at_oracle_sizes(ctx, name):
    """bench.py's configs[2] / configs[4] constructions (recompressed plates x jittered plates;
    complex Helmholtz on the Fibonacci sphere with orders growing per level, recompressed at
    1e-4) at N = 4096, against the oracle and the dense product."""
    import bench
    _, _, _, A, B = bench.build_operands(name, 4096)
    eps = bench.CONFIGS[name][3]
    got, ref, cg, co = check_against_oracle(A, B, eps, ctx)
    dense = O.h2_to_dense(A) @ O.h2_to_dense(B)
    assert rel(cg, dense) <= 1.1 * rel(co, dense) + 1e-13
    if name == "cfg5":
        assert A.scalar == P.H2C_COMPLEX


# ---- exact H^2 MVP on the device (h2_matrix.cpp:213-278) and eps_rel (metrics.cpp:37-55)
@pytest.mark.parametrize("kind", ["real", "complex"])
def test_mvp_matches_oracle(ctx, kind):
    if kind == "real":
        A = laplace(1024, 5, 16, 1.2)
    else:
        _, _, A = helmholtz(3, 20, 1.5)
    n = A.size()
    X = np.stack([P.random_vector(n, s_, kind == "complex") for s_ in range(3)], 1)
    Y = P.mvp(A, X, ctx)
    for j in range(3):
        ref = O.mvp(A, X[:, j])
        assert np.linalg.norm(Y[:, j] - ref) <= 1e-13 * np.linalg.norm(ref)
    y1 = P.mvp(A, X[:, 0], ctx)
    assert np.linalg.norm(y1 - O.mvp(A, X[:, 0])) <= 1e-13 * np.linalg.norm(y1)


@pytest.mark.parametrize("kind", ["real", "complex", "product"])
def test_device_h2_to_dense_matches_oracle(ctx, kind):
    """h2_to_dense on the device (A * I through the MVP, h2_matrix.cpp:124-137) vs the oracle's block sum."""
    if kind == "real":
        A = laplace(1024, 5, 16, 1.2)
    elif kind == "complex":
        _, _, A = helmholtz(3, 20, 1.5)
    else:
        B = chebyshev(4096, 32, 3)
        A = P.mmp(B, B, 1e-6, ctx).product
    D = P.h2_to_dense(A, ctx)
    ref = O.h2_to_dense(A)
    assert D.shape == ref.shape and D.dtype == ref.dtype
    assert rel(D, ref) <= 1e-14


def test_relative_error_matches_oracle(ctx):
    A = chebyshev(4096, 32, 3)
    C = P.mmp(A, A, 1e-6, ctx).product
    e_gpu = P.relative_error(A, A, C, 99, ctx)
    e_ora = O.relative_error(A, A, C, 99)
    assert abs(e_gpu - e_ora) <= 1e-9 * max(e_ora, 1e-30) + 1e-15


# ---- the device truncation (truncation.cpp:9-47) on the reference's KATs and random Grams
def test_device_truncation_known_answers(ctx):
    assert P.svd_truncate_gram(np.eye(4), 1e-2, ctx)[0].shape[1] == 4
    assert P.svd_truncate_gram(np.diag([1.0, 1e-1, 1e-3, 0.0]), 1e-2, ctx)[0].shape[1] == 2
    tie = np.diag([1.0, 1e-2])
    assert P.svd_truncate_gram(tie, 1e-2, ctx)[0].shape[1] == 1
    assert P.svd_truncate_gram(tie, 0.5e-2, ctx)[0].shape[1] == 2
    b, dg = P.svd_truncate_gram(np.zeros((5, 5)), 1e-4, ctx)
    assert dg and b.shape == (5, 1) and b[0, 0] == 1.0 and np.all(b[1:] == 0)
    with pytest.raises(P.ConfigError):
        P.svd_truncate_gram(np.eye(3), 1.0, ctx)


@pytest.mark.parametrize("n", [6, 33, 64, 100, 150, 224, 300, 480, 610, 700])
@pytest.mark.parametrize("cplx", [False, True])
def test_device_truncation_matches_oracle(ctx, n, cplx):
    """heev_kernel (one cluster per Gram: 1..16 CTAs, global slabs beyond) against LAPACK."""
    rng = np.random.default_rng(n)
    k = max(1, (2 * n) // 3)
    m = rng.standard_normal((n, k)) * np.logspace(0, -9, k)
    if cplx:
        m = m + 1j * rng.standard_normal((n, k)) * np.logspace(0, -9, k)
    g = m @ m.conj().T
    for eps in (1e-4, 1e-8):
        bg, dg = P.svd_truncate_gram(g, eps, ctx)
        bo, do = O.svd_truncate_gram(g, eps)
        assert bg.shape == bo.shape and dg == do
        assert np.abs(bg.conj().T @ bg - np.eye(bg.shape[1])).max() <= 1e-12
        # same subspace: projector difference
        assert np.linalg.norm(bg @ bg.conj().T - bo @ bo.conj().T) <= 1e-6


@pytest.mark.parametrize("cplx", [False, True])
def test_device_truncation_clustered_spectrum(ctx, cplx):
    """Exactly repeated eigenvalues (identity-like Grams, as the square leaf bases of configs[1]
    give: G3 = V V^H = I) and a degenerate tail: same rank, orthonormal kept basis spanning the
    oracle's dominant subspace."""
    rng = np.random.default_rng(7)
    for n, k in ((64, 20), (128, 50), (200, 64)):
        m = rng.standard_normal((n, k)) + (1j * rng.standard_normal((n, k)) if cplx else 0)
        q, _ = np.linalg.qr(m)
        g = 0.125 * np.eye(n) + q @ np.diag(np.repeat([1.0, 0.5], k // 2)) @ q.conj().T
        for eps in (1e-4, 0.5):
            bg, dg = P.svd_truncate_gram(g, eps, ctx)
            bo, do = O.svd_truncate_gram(g, eps)
            assert bg.shape == bo.shape and dg == do
            assert np.abs(bg.conj().T @ bg - np.eye(bg.shape[1])).max() <= 1e-12
            assert np.linalg.norm(bg @ bg.conj().T - bo @ bo.conj().T) <= 1e-10
