"""CPU checks of bench.py's synthetic BASELINE inputs: the geometries have
the configured sizes and spacings, the Helmholtz orders grow with the box size, and the constructed
operands of every config are valid H^2 matrices over the shared structure at a small N."""
import numpy as np
import pytest

import bench
import paper_1908_05218_b200 as P


def test_plate_geometry():
    pts, h = bench.plate_points(262144)
    assert pts.shape == (262144, 3) and h == pytest.approx(1 / 128)
    z = np.unique(np.round(pts[:, 2], 12))
    assert np.allclose(z, 0.1 * np.arange(16))
    xs = np.unique(np.round(pts[:, 0], 12))
    assert len(xs) == 128 and np.allclose(np.diff(xs), h)


def test_sphere_geometry_fixed_points_per_wavelength():
    for n in (4096, 65536):
        x = bench.sphere_points(n)
        r = np.linalg.norm(x, axis=1)
        assert np.allclose(r, 8.0 * np.sqrt(n / 2 ** 20))
    # full size: diameter 16 wavelengths (kappa = 2 pi)
    assert 2 * 8.0 * bench.KAPPA / (2 * np.pi) == 16.0


def test_helmholtz_orders_grow_toward_the_root():
    x = bench.sphere_points(65536)
    t = P.build_cluster_tree(x, 64)
    o = bench.helmholtz_orders(t)
    assert o.shape == (t.depth + 1,)
    assert (np.diff(o) <= 0).all() and o[-1] == 3 and o.max() <= bench.HELM_ORDER_CAP and o.max() > 5


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_bench_operands_small(name):
    pts, t, s, A, B = bench.build_operands(name, 4096 if name != "cfg4" else 4096)
    assert A.tree is t and B.tree is t and A.structure is s and B.structure is s
    for M in (A, B):
        for c in range(t.n_clusters):
            if t.parent[c] < 0:
                continue
            v = M.row_basis(c)
            assert np.abs(v.conj().T @ v - np.eye(M.row_rank[c])).max() < 1e-11
    if name == "cfg5":
        assert A.scalar == P.H2C_COMPLEX and B is A
    if name in ("cfg3", "cfg4"):
        assert B is not A


def _recompression_case(kind):
    from oracle import pyoracle as O  # checker only
    if kind == "helmholtz":
        n, leaf, eps = 4096, 64, 1e-4
        pts = bench.sphere_points(n) * 0.5  # ~4 wavelengths across
    else:
        n, leaf, eps = 4096, 32, 1e-6
        pts = O.geometry("random_cloud", seed=1, n=n)
    t = O.build_cluster_tree(pts, leaf)
    s = O.build_block_tree(t, 1.0)
    orders = bench.helmholtz_orders(t, hi=7) if kind == "helmholtz" else 4
    kap = bench.KAPPA if kind == "helmholtz" else 0.0
    A0 = P.build_chebyshev(t, s, pts, orders, kernel=kind, kappa=kap)
    Ar = P.build_chebyshev(t, s, pts, orders, kernel=kind, kappa=kap, eps_recompress=eps)
    D0 = O.h2_to_dense(A0)
    Aref = O.build_h2(D0, s, eps)  # the reference's rule (h2_matrix.cpp:83-181) on the dense operand
    return O, D0, Ar, Aref


def _check_recompression(kind):
    O, D0, Ar, Aref = _recompression_case(kind)
    assert np.array_equal(Ar.row_rank, Aref.row_rank) and np.array_equal(Ar.col_rank, Aref.col_rank)
    assert np.array_equal(Ar.row_degenerate, Aref.row_degenerate)
    Dr, Dref = O.h2_to_dense(Ar), O.h2_to_dense(Aref)
    assert np.linalg.norm(Dr - Dref) <= 1e-11 * np.linalg.norm(D0)


@pytest.mark.parametrize("kind", ["laplace", "helmholtz"])
def test_recompression_matches_the_reference_rule(kind):
    """The constructor's recompression (construct.cpp, host path here) equals the reference's own
    build_h2 (oracle restatement, pinned to the reference by tests/test_ref_golden.py) applied to
    the dense interpolation operand: equal ranks, same matrix to round-off."""
    _check_recompression(kind)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["laplace", "helmholtz"])
def test_device_recompression_matches_the_reference_rule(kind):
    """Same with the constructor's device passes (construct_dev.cu) active."""
    _check_recompression(kind)
