"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_build/liboracle.so, the CPU restatement of the
reference's MMP path.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs import this module, and only as the checker; the product
package never does.  It reuses the product's descriptor structs so both sides
see the very same buffers.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_1908_05218_b200.h2c import (BlockTree, ClusterTree, ConfigError, H2Matrix, InvariantError, MmpReport,
                                       MmpResult, P_f64, P_i32, P_i64, h2c_blocks, h2c_matrix, h2c_report, h2c_tree,
                                       H2C_COMPLEX, H2C_REAL)

LIBPATH = Path(__file__).resolve().parent / "_build" / "liboracle.so"
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIBPATH.exists():
            raise ImportError(f"{LIBPATH} missing: run `make -C oracle`")
        L = C.CDLL(str(LIBPATH))
        L.h2o_last_error.restype = C.c_char_p
        L.h2o_set_threads.argtypes = [C.c_int]
        L.h2o_geometry_count.restype = C.c_int64
        L.h2o_geometry_count.argtypes = [C.c_int, C.c_uint64] + [C.c_int] * 7
        L.h2o_geometry_fill.restype = C.c_int
        L.h2o_geometry_fill.argtypes = [C.c_int, C.c_uint64] + [C.c_int] * 7 + [P_f64]
        L.h2o_assemble_dense.restype = C.c_int
        L.h2o_assemble_dense.argtypes = [P_f64, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, P_f64]
        L.h2o_build_tree.restype = C.c_void_p
        L.h2o_build_tree.argtypes = [P_f64, C.c_int, C.c_int]
        L.h2o_tree_desc.argtypes = [C.c_void_p, C.POINTER(h2c_tree)]
        L.h2o_tree_free.argtypes = [C.c_void_p]
        L.h2o_build_blocks.restype = C.c_void_p
        L.h2o_build_blocks.argtypes = [C.POINTER(h2c_tree), C.c_double]
        L.h2o_blocks_desc.argtypes = [C.c_void_p, C.POINTER(h2c_blocks)]
        L.h2o_blocks_free.argtypes = [C.c_void_p]
        L.h2o_target_status.restype = C.c_int
        L.h2o_target_status.argtypes = [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), C.c_int, C.c_int]
        L.h2o_build_h2.restype = C.c_void_p
        L.h2o_build_h2.argtypes = [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), C.c_int, P_f64, C.c_double]
        L.h2o_matrix_desc.argtypes = [C.c_void_p, C.POINTER(h2c_matrix)]
        L.h2o_matrix_free.argtypes = [C.c_void_p]
        L.h2o_truncate_gram.restype = C.c_int
        L.h2o_truncate_gram.argtypes = [C.c_int, P_f64, C.c_int, C.c_double, P_f64, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]
        L.h2o_mmp.restype = C.c_int
        L.h2o_mmp.argtypes = [C.POINTER(h2c_matrix), C.POINTER(h2c_matrix), C.c_double, C.c_int, C.c_int64,
                              C.POINTER(C.c_void_p)]
        L.h2o_result_matrix.argtypes = [C.c_void_p, C.POINTER(h2c_matrix)]
        L.h2o_result_report.argtypes = [C.c_void_p, C.POINTER(h2c_report)]
        L.h2o_result_min_margin.restype = C.c_double
        L.h2o_result_min_margin.argtypes = [C.c_void_p]
        L.h2o_result_free.argtypes = [C.c_void_p]
        L.h2o_basis_products.restype = C.c_int64
        L.h2o_basis_products.argtypes = [C.POINTER(h2c_matrix), C.POINTER(h2c_matrix), P_i64, P_i32, P_i32, P_f64,
                                         C.c_int64]
        L.h2o_h2_to_dense.restype = C.c_int
        L.h2o_h2_to_dense.argtypes = [C.POINTER(h2c_matrix), P_f64]
        L.h2o_mvp.restype = C.c_int
        L.h2o_mvp.argtypes = [C.POINTER(h2c_matrix), P_f64, P_f64]
        L.h2o_memory_footprint.restype = C.c_int64
        L.h2o_memory_footprint.argtypes = [C.POINTER(h2c_matrix)]
        L.h2o_random_vector.restype = C.c_int
        L.h2o_random_vector.argtypes = [C.c_int, C.c_uint64, C.c_int, P_f64]
        L.h2o_relative_error.restype = C.c_int
        L.h2o_relative_error.argtypes = [C.POINTER(h2c_matrix)] * 3 + [C.c_uint64, C.POINTER(C.c_double),
                                                                        C.POINTER(C.c_int)]
        L.h2o_set_mmp_threads.argtypes = [C.c_int]
        L.h2o_mvp_multi.restype = C.c_int
        L.h2o_mvp_multi.argtypes = [C.POINTER(h2c_matrix), P_f64, C.c_int, P_f64]
        L.h2o_sliced_start.restype = C.c_void_p
        L.h2o_sliced_start.argtypes = [C.POINTER(h2c_matrix), C.POINTER(h2c_matrix), C.c_double, C.c_int, C.c_int]
        L.h2o_sliced_step.restype = C.c_int
        L.h2o_sliced_step.argtypes = [C.c_void_p, C.c_double, C.POINTER(C.c_double), P_i64, P_i64]
        L.h2o_sliced_stop.argtypes = [C.c_void_p]
        L.h2o_set_threads(1)
        _lib = L
    return _lib


def _err() -> str:
    m = lib().h2o_last_error()
    return m.decode() if m else ""


def _check(rc: int) -> None:
    if rc == 0:
        return
    if rc == 2:
        raise ConfigError(_err())
    raise InvariantError(_err())


FAMILY = {"random_cloud": 0, "bus": 1, "slab": 2, "cube_array": 3}


def geometry(family: str = "random_cloud", seed: int = 0, n: int = 0, bus_count: int = 0, samples_per_meter: int = 1,
             slab_width: int = 0, slab_thickness: int = 2, array_edge: int = 0, cube_points: int = 3) -> np.ndarray:
    """generate_geometry (geometry.cpp:159-181)."""
    args = (FAMILY[family], seed, n, bus_count, samples_per_meter, slab_width, slab_thickness, array_edge, cube_points)
    cnt = lib().h2o_geometry_count(*args)
    if cnt < 0:
        raise ConfigError(_err())
    out = np.zeros((cnt, 3))
    _check(lib().h2o_geometry_fill(*args, out.ctypes.data_as(P_f64)))
    return out


def assemble_dense(points: np.ndarray, kernel: str = "laplace", wavenumber: float = 0.0, diagonal=None) -> np.ndarray:
    """assemble_dense (geometry.cpp:200-233): 1/r or exp(ikr)/r, original ordering."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = len(pts)
    cplx = kernel == "helmholtz"
    out = np.zeros((n, n), dtype=np.complex128 if cplx else np.float64, order="F")
    _check(lib().h2o_assemble_dense(pts.ctypes.data_as(P_f64), n, int(cplx), wavenumber, diagonal is not None,
                                    0.0 if diagonal is None else float(diagonal), out.ctypes.data_as(P_f64)))
    return out


def build_cluster_tree(points: np.ndarray, leafsize: int) -> ClusterTree:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    h = lib().h2o_build_tree(pts.ctypes.data_as(P_f64), len(pts), leafsize)
    if not h:
        raise ConfigError(_err())
    try:
        d = h2c_tree()
        lib().h2o_tree_desc(h, C.byref(d))
        t = ClusterTree.from_desc(d)
        t.points = pts
        return t
    finally:
        lib().h2o_tree_free(h)


def build_block_tree(tree: ClusterTree, eta: float) -> BlockTree:
    h = lib().h2o_build_blocks(C.byref(tree.desc()), eta)
    if not h:
        raise ConfigError(_err())
    try:
        d = h2c_blocks()
        lib().h2o_blocks_desc(h, C.byref(d))
        return BlockTree.from_desc(tree, d)
    finally:
        lib().h2o_blocks_free(h)


def target_status(structure: BlockTree, t: int, s: int) -> int:
    r = lib().h2o_target_status(C.byref(structure.tree.desc()), C.byref(structure.desc()), t, s)
    if r < 0:
        raise InvariantError(_err())
    return r


def build_h2(dense: np.ndarray, structure: BlockTree, eps_h2: float) -> H2Matrix:
    """build_h2 (h2_matrix.cpp:141-181), dense in the original ordering."""
    cplx = np.iscomplexobj(dense)
    d = np.asfortranarray(dense, dtype=np.complex128 if cplx else np.float64)
    h = lib().h2o_build_h2(C.byref(structure.tree.desc()), C.byref(structure.desc()), int(cplx),
                           d.ctypes.data_as(P_f64), eps_h2)
    if not h:
        raise ConfigError(_err())
    try:
        md = h2c_matrix()
        lib().h2o_matrix_desc(h, C.byref(md))
        return H2Matrix.from_desc(structure.tree, structure, md)
    finally:
        lib().h2o_matrix_free(h)


def svd_truncate_gram(gram: np.ndarray, eps: float):
    """svd_truncate_gram (truncation.cpp:9-47) -> (basis, degenerate)."""
    g = np.asfortranarray(gram)
    cplx = np.iscomplexobj(g)
    if g.ndim != 2 or g.shape[0] != g.shape[1] or g.shape[0] < 1:
        raise ConfigError("svd_truncate_gram: gram matrix must be square and non-empty")
    n = g.shape[0]
    basis = np.zeros((n, n), dtype=g.dtype, order="F")
    rank, degen = C.c_int(), C.c_int()
    _check(lib().h2o_truncate_gram(int(cplx), g.ctypes.data_as(P_f64), n, eps, basis.ctypes.data_as(P_f64),
                                   C.byref(rank), C.byref(degen)))
    return basis[:, :rank.value].copy(), bool(degen.value)


def mmp(a: H2Matrix, b: H2Matrix, eps: float, adaptive: bool = True, ff_cache_bytes: int = 8 << 30,
        with_margin: bool = False, threads: int = 1):
    """mmp / formatted_mmp of the CPU oracle (mmp.cpp:688-719).  threads > 1 runs the
    parallel restatement (bit-identical result, oracle/product_engine.cpp)."""
    out = C.c_void_p()
    lib().h2o_set_mmp_threads(int(threads))
    _check(lib().h2o_mmp(C.byref(a.desc()), C.byref(b.desc()), eps, int(adaptive), ff_cache_bytes, C.byref(out)))
    try:
        d = h2c_matrix()
        lib().h2o_result_matrix(out, C.byref(d))
        prod = H2Matrix.from_desc(a.tree, a.structure, d)
        r = h2c_report()
        lib().h2o_result_report(out, C.byref(r))
        rep = MmpReport.from_desc(r)
        margin = lib().h2o_result_min_margin(out)
    finally:
        lib().h2o_result_free(out)
    res = MmpResult(prod, rep)
    return (res, margin) if with_margin else res


def formatted_mmp(a: H2Matrix, b: H2Matrix) -> MmpResult:
    return mmp(a, b, 0.0, adaptive=False)


def basis_products(a: H2Matrix, b: H2Matrix) -> list:
    nc = a.tree.n_clusters
    offs = np.zeros(nc, dtype=np.int64)
    rows = np.zeros(nc, dtype=np.int32)
    cols = np.zeros(nc, dtype=np.int32)
    need = lib().h2o_basis_products(C.byref(a.desc()), C.byref(b.desc()), offs.ctypes.data_as(P_i64),
                                    rows.ctypes.data_as(P_i32), cols.ctypes.data_as(P_i32), None, 0)
    if need < 0:
        raise ConfigError(_err())
    vals = np.zeros(max(1, need), dtype=a.dtype)
    lib().h2o_basis_products(C.byref(a.desc()), C.byref(b.desc()), offs.ctypes.data_as(P_i64),
                             rows.ctypes.data_as(P_i32), cols.ctypes.data_as(P_i32), vals.ctypes.data_as(P_f64), need)
    return [vals[offs[i]:offs[i] + rows[i] * cols[i]].reshape(cols[i], rows[i]).T for i in range(nc)]


def h2_to_dense(m: H2Matrix) -> np.ndarray:
    n = m.tree.n_points
    out = np.zeros((n, n), dtype=m.dtype, order="F")
    _check(lib().h2o_h2_to_dense(C.byref(m.desc()), out.ctypes.data_as(P_f64)))
    return out


def mvp(m: H2Matrix, x: np.ndarray) -> np.ndarray:
    xx = np.ascontiguousarray(x, dtype=m.dtype)
    y = np.zeros_like(xx)
    _check(lib().h2o_mvp(C.byref(m.desc()), xx.ctypes.data_as(P_f64), y.ctypes.data_as(P_f64)))
    return y


def mvp_multi(m: H2Matrix, x: np.ndarray, threads: int = 1) -> np.ndarray:
    """Y = A X for the columns of X (N x nv), the columns on `threads` threads."""
    xx = np.asfortranarray(x, dtype=m.dtype)
    if xx.ndim == 1:
        xx = xx.reshape(-1, 1, order="F")
    y = np.zeros_like(xx)
    lib().h2o_set_mmp_threads(int(threads))
    _check(lib().h2o_mvp_multi(C.byref(m.desc()), xx.ctypes.data_as(P_f64), xx.shape[1], y.ctypes.data_as(P_f64)))
    return y


class SlicedProduct:
    """Consecutive slices of all-cores oracle products C = A*B (bench.py's CPU
    baseline): step(seconds) lets the engine run that long, returns at its next
    slice point with (wall seconds, reference MACs counted in the slice, products
    completed so far).  Products run back to back while steps are requested."""

    def __init__(self, a: H2Matrix, b: H2Matrix, eps: float, threads: int, adaptive: bool = True):
        self._a, self._b = a, b  # the descriptors must outlive the engine
        self._h = lib().h2o_sliced_start(C.byref(a.desc()), C.byref(b.desc()), eps, int(adaptive), int(threads))
        if not self._h:
            raise ConfigError(_err())

    def step(self, seconds: float):
        el, macs, prods = C.c_double(), C.c_int64(), C.c_int64()
        _check(lib().h2o_sliced_step(self._h, seconds, C.byref(el), C.byref(macs), C.byref(prods)))
        return el.value, int(macs.value), int(prods.value)

    def close(self) -> None:
        if self._h:
            lib().h2o_sliced_stop(self._h)
            self._h = None

    def __del__(self):
        self.close()


def memory_footprint(m: H2Matrix) -> int:
    return int(lib().h2o_memory_footprint(C.byref(m.desc())))


def random_vector(n: int, seed: int, complex_: bool = False) -> np.ndarray:
    out = np.zeros(n, dtype=np.complex128 if complex_ else np.float64)
    _check(lib().h2o_random_vector(n, seed, int(complex_), out.ctypes.data_as(P_f64)))
    return out


def relative_error(a: H2Matrix, b: H2Matrix, c: H2Matrix, seed: int) -> float:
    v, z = C.c_double(), C.c_int()
    _check(lib().h2o_relative_error(C.byref(a.desc()), C.byref(b.desc()), C.byref(c.desc()), seed, C.byref(v),
                                    C.byref(z)))
    return v.value
