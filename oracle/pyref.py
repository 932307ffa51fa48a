"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_ref/libh2ref.so: the REFERENCE's own MMP-path sources
(/root/reference/proj/core/src, unmodified) compiled here against
oracle/eigen_shim (Eigen is absent from this image), driven by
oracle/ref_driver.cpp.  Used by tools/make_ref_golden.py (writes
tests/golden/ref_cases.npz, here) and by bench.py's reference arm
(`--impl reference`: SlicedReference times the reference's own mmp() on the
bench workload).  The prebuilt .so travels to the GPU box with the snapshot;
/root/reference itself is never read at run time.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_1908_05218_b200.h2c import P_f64, h2c_blocks, h2c_matrix, h2c_report, h2c_tree

LIBPATH = Path(__file__).resolve().parent / "_ref" / "libh2ref.so"
FAMILIES = {"random_cloud": 0, "bus": 1, "slab": 2, "cube_array": 3}
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIBPATH.exists():
            raise ImportError(f"{LIBPATH} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(str(LIBPATH))
        L.h2r_last_error.restype = C.c_char_p
        L.h2r_run.restype = C.c_void_p
        L.h2r_run.argtypes = ([C.c_int, C.c_uint64] + [C.c_int] * 8 + [C.c_double, C.c_int, C.c_double, C.c_int]
                              + [C.c_double] * 3 + [C.c_int, C.POINTER(C.c_int)])
        L.h2r_tree.argtypes = [C.c_void_p, C.POINTER(h2c_tree)]
        L.h2r_blocks.argtypes = [C.c_void_p, C.POINTER(h2c_blocks)]
        L.h2r_matrix.argtypes = [C.c_void_p, C.c_int, C.POINTER(h2c_matrix)]
        L.h2r_report.argtypes = [C.c_void_p, C.POINTER(h2c_report)]
        L.h2r_mvp.argtypes = [C.c_void_p, C.c_int, P_f64, C.c_int, P_f64]
        L.h2r_relative_error.restype = C.c_double
        L.h2r_relative_error.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
        L.h2r_truncate_gram.argtypes = [C.c_int, P_f64, C.c_int, C.c_double, P_f64, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]
        L.h2r_free.argtypes = [C.c_void_p]
        L.h2r_shape_mismatches.restype = C.c_longlong
        L.h2r_sliced_start.restype = C.c_void_p
        L.h2r_sliced_start.argtypes = [C.POINTER(h2c_matrix), C.POINTER(h2c_matrix), C.c_double, C.c_int,
                                       C.POINTER(C.c_int)]
        L.h2r_sliced_step.argtypes = [C.c_void_p, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.h2r_sliced_stop.argtypes = [C.c_void_p]
        L.h2r_mac_counter.restype = C.c_longlong
        _lib = L
    return _lib


def _arr(ptr, n, dtype):
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True) if n else np.zeros(0, dtype)


class RefCase:
    """One run of the reference pipeline: geometry -> trees -> dense -> build_h2 -> mmp."""

    def __init__(self, family="random_cloud", seed=0, n=0, bus_count=0, samples_per_meter=1, slab_width=0,
                 slab_thickness=2, array_edge=0, cube_points=3, leafsize=30, eta=1.0, kernel="laplace",
                 wavenumber=0.0, diagonal=None, eps_h2=1e-4, eps=1e-6, mode="mmp"):
        code = C.c_int(0)
        m = {"mmp": 0, "formatted": 1, "build": 2}[mode]
        self.h = lib().h2r_run(FAMILIES[family], seed, n, bus_count, samples_per_meter, slab_width, slab_thickness,
                               array_edge, cube_points, leafsize, eta, int(kernel == "helmholtz"), wavenumber,
                               int(diagonal is not None), float(diagonal or 0.0), eps_h2, eps, m, C.byref(code))
        if not self.h:
            raise RuntimeError(f"reference error {code.value}: {lib().h2r_last_error().decode()}")
        self.cplx = kernel == "helmholtz"
        t = h2c_tree()
        lib().h2r_tree(self.h, C.byref(t))
        b = h2c_blocks()
        lib().h2r_blocks(self.h, C.byref(b))
        self.n = t.n_points
        self.tree = {"depth": t.depth, "perm": _arr(t.perm, t.n_points, np.int32),
                     "begin": _arr(t.begin, t.n_clusters, np.int32), "end": _arr(t.end, t.n_clusters, np.int32),
                     "parent": _arr(t.parent, t.n_clusters, np.int32)}
        self.blocks = {"c_sp": b.c_sp, "level_ptr": _arr(b.level_ptr, b.depth + 2, np.int64),
                       "row": _arr(b.row, b.n_blocks, np.int32), "col": _arr(b.col, b.n_blocks, np.int32),
                       "kind": _arr(b.kind, b.n_blocks, np.uint8)}
        self.nc = t.n_clusters
        self.mode = mode

    def ranks(self, which):
        d = h2c_matrix()
        lib().h2r_matrix(self.h, which, C.byref(d))
        return (_arr(d.row_rank, self.nc, np.int32), _arr(d.col_rank, self.nc, np.int32),
                _arr(d.row_degenerate, self.nc, np.uint8), _arr(d.col_degenerate, self.nc, np.uint8))

    def report(self):
        r = h2c_report()
        if lib().h2r_report(self.h, C.byref(r)):
            raise RuntimeError("no product")
        nl = r.n_levels
        return {"flops": r.flops, "case_flops": np.array(r.case_flops[:4], np.int64),
                "max_row_rank": _arr(r.max_row_rank, nl, np.int64), "max_col_rank": _arr(r.max_col_rank, nl, np.int64),
                "case_products": _arr(r.case_products, 4 * nl, np.int64).reshape(nl, 4),
                "max_case1_terms": _arr(r.max_case1_terms, nl, np.int32),
                "max_case2_terms": _arr(r.max_case2_terms, nl, np.int32),
                "max_case3_terms": _arr(r.max_case3_terms, nl, np.int32),
                "pending_after_split": r.pending_after_split, "wall_seconds": r.wall_seconds}

    def mvp(self, which, X):
        """Y = M X (M = A for which=0, C for which=1), X: N x nv (complex for Helmholtz)."""
        X = np.asfortranarray(X, dtype=np.complex128 if self.cplx else np.float64)
        nv = X.shape[1]
        xf = np.ascontiguousarray(X.T).view(np.float64).ravel()
        y = np.zeros_like(xf)
        if lib().h2r_mvp(self.h, which, xf.ctypes.data_as(P_f64), nv, y.ctypes.data_as(P_f64)):
            raise RuntimeError(lib().h2r_last_error().decode())
        Y = y.view(np.complex128 if self.cplx else np.float64).reshape(nv, self.n).T
        return Y

    def relative_error(self, seed):
        z = C.c_int(0)
        return lib().h2r_relative_error(self.h, seed, C.byref(z))

    def __del__(self):
        if getattr(self, "h", None):
            lib().h2r_free(self.h)
            self.h = None


def shape_mismatches() -> int:
    return lib().h2r_shape_mismatches()


def available() -> bool:
    return LIBPATH.exists()


class SlicedReference:
    """The reference's own mmp() (single-threaded, mmp.hpp:58-66) run back to back on operands given
    as flat descriptors (converted into the reference's types, block tree rebuilt by the reference
    and checked against the descriptor's).  step(seconds) -> (wall seconds, reference MACs in the
    window — the shim counts exactly MmpReport.flops' rule —, products completed, their flops)."""

    def __init__(self, a, b, eps: float, adaptive: bool = True):
        self._a, self._b = a, b  # the descriptors must outlive the engine
        self._da, self._db = a.desc(), b.desc()
        code = C.c_int(0)
        self._h = lib().h2r_sliced_start(C.byref(self._da), C.byref(self._da) if b is a else C.byref(self._db),
                                         eps, int(adaptive), C.byref(code))
        if not self._h:
            raise RuntimeError(f"reference error {code.value}: {lib().h2r_last_error().decode()}")

    def step(self, seconds: float):
        el, macs, prods, pf = C.c_double(), C.c_int64(), C.c_int64(), C.c_int64()
        if lib().h2r_sliced_step(self._h, seconds, C.byref(el), C.byref(macs), C.byref(prods), C.byref(pf)):
            raise RuntimeError(lib().h2r_last_error().decode())
        return el.value, int(macs.value), int(prods.value), int(pf.value)

    def close(self) -> None:
        if self._h:
            lib().h2r_sliced_stop(self._h)
            self._h = None

    def __del__(self):
        self.close()
