"""Python mirror of the reference's public MMP API (proj/core/include/h2mmp):

    build_cluster_tree(points, leafsize)          cluster_tree.hpp:43
    build_block_tree(rows, cols, eta)             block_tree.hpp:75-77
    mmp(a, b, eps_trunc) -> MmpResult             mmp.hpp:60-61
    formatted_mmp(a, b) -> MmpResult              mmp.hpp:66-67

plus the synthetic-input constructors of the BASELINE configs.  Every call
goes through the C-ABI of libh2mmp_b200.so; the product runs on the GPU only.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional

import numpy as np

from . import h2c
from .h2c import (BlockTree, ClusterTree, ConfigError, H2Matrix, MmpReport, MmpResult, h2c_blocks, h2c_matrix,
                  h2c_report, h2c_tree, raise_for)

_ctx_lock = threading.Lock()
_default_ctx: Optional["Context"] = None


class Context:
    """A device, a CUDA stream and the structure-plan cache (h2c_create)."""

    def __init__(self, device: int = 0):
        self._h = h2c.lib().h2c_create(device)
        if not self._h:
            raise h2c.DeviceError(h2c.last_error())

    @property
    def handle(self):
        return self._h

    def kernel_launches(self) -> int:
        return int(h2c.lib().h2c_kernel_launches(self._h))

    def stream_ptr(self) -> int:
        """cudaStream_t of the library (for torch.cuda.ExternalStream events)."""
        return int(h2c.lib().h2c_stream(self._h) or 0)

    def set_profile(self, on: bool) -> None:
        h2c.lib().h2c_set_profile(self._h, int(on))

    def profile(self) -> list[dict]:
        """Per (phase/kernel) CUDA-event totals of the last call."""
        L = h2c.lib()
        out = []
        for i in range(L.h2c_profile_count(self._h)):
            name = C.create_string_buffer(128)
            n, ms, macs = C.c_int64(), C.c_double(), C.c_int64()
            L.h2c_profile_get(self._h, i, name, 128, C.byref(n), C.byref(ms), C.byref(macs))
            out.append({"name": name.value.decode(), "launches": n.value, "ms": ms.value, "macs": macs.value,
                        "bytes": int(L.h2c_profile_bytes(self._h, i))})
        return out

    def close(self):
        if self._h:
            h2c.lib().h2c_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_context() -> Context:
    global _default_ctx
    with _ctx_lock:
        if _default_ctx is None:
            _default_ctx = Context(0)
        return _default_ctx


# ---------------------------------------------------------------------------
def _structure(points: np.ndarray, leafsize: int, eta: float):
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    L = h2c.lib()
    h = L.h2c_build_structure(pts.ctypes.data_as(h2c.P_f64), len(pts), int(leafsize), float(eta))
    if not h:
        msg = h2c.last_error()
        raise ConfigError(msg) if ("must" in msg or "cannot" in msg) else h2c.InvariantError(msg)
    try:
        td, bd = h2c_tree(), h2c_blocks()
        L.h2c_structure_tree(h, C.byref(td))
        L.h2c_structure_blocks(h, C.byref(bd))
        tree = ClusterTree.from_desc(td)
        tree.points = pts
        blocks = BlockTree.from_desc(tree, bd)
    finally:
        L.h2c_structure_free(h)
    return tree, blocks


def build_cluster_tree(points: np.ndarray, leafsize: int) -> ClusterTree:
    """cluster_tree.cpp:66-93 (longest-axis median bisection to uniform depth)."""
    tree, _ = _structure(points, leafsize, 1.0)
    return tree


def build_block_tree(rows: ClusterTree, cols: ClusterTree, eta: float) -> BlockTree:
    """block_tree.cpp:9-53; the MMP path uses a single shared tree (rows is cols)."""
    if rows is not cols:
        raise ConfigError("build_block_tree: the B200 path requires one shared cluster tree")
    if eta <= 0:
        raise ConfigError("eta must be positive")
    if rows.points is None:
        raise ConfigError("build_block_tree: tree was not built from points")
    t2, blocks = _structure(rows.points, rows.leafsize, eta)
    if not t2.same_as(rows):
        raise h2c.InvariantError("block tree rebuilt a different cluster tree")
    blocks.tree = rows
    return blocks


def target_status(structure: BlockTree, t: int, s: int) -> int:
    """BlockTree::target_status (block_tree.cpp:61-85): 0 full, 1 adm, 2 sub, 3 inside."""
    r = h2c.lib().h2c_target_status(C.byref(structure.tree.desc()), C.byref(structure.desc()), int(t), int(s))
    if r < 0:
        raise h2c.InvariantError(h2c.last_error())
    return r


def _take_h2(handle, tree: ClusterTree, structure: BlockTree) -> H2Matrix:
    L = h2c.lib()
    if not handle:
        raise ConfigError(h2c.last_error())
    try:
        d = h2c_matrix()
        L.h2c_h2_desc(handle, C.byref(d))
        return H2Matrix.from_desc(tree, structure, d)
    finally:
        L.h2c_h2_free(handle)


def random_cloud(n: int, seed: int) -> np.ndarray:
    """make_random_cloud (geometry.cpp:39-52): [n, 3] points uniform in the unit cube."""
    out = np.zeros((int(n), 3))
    raise_for(h2c.lib().h2c_random_cloud(int(n), int(seed), out.ctypes.data_as(h2c.P_f64)), h2c.last_error())
    return out


def build_chebyshev(tree: ClusterTree, structure: BlockTree, points: np.ndarray, order, kernel: str = "laplace",
                    kappa: float = 0.0, diagonal: float = 0.0, eps_recompress: float = 0.0,
                    threads: int = 0) -> H2Matrix:
    """Nested tensor-Chebyshev H^2 matrix with orthonormal bases (input side).

    order: one interpolation order, or one per tree level (depth + 1 entries).
    eps_recompress > 0: recompress with the reference's build_h2 rule (h2_matrix.cpp:83-121)."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    k = {"laplace": 0, "helmholtz": 1}[kernel]
    if np.ndim(order) == 0:
        orders = np.full(tree.depth + 1, int(order), dtype=np.int32)
    else:
        orders = np.ascontiguousarray(order, dtype=np.int32)
        if orders.shape != (tree.depth + 1,):
            raise ConfigError(f"orders must have depth + 1 = {tree.depth + 1} entries")
    h = h2c.lib().h2c_build_chebyshev_orders(C.byref(tree.desc()), C.byref(structure.desc()),
                                             pts.ctypes.data_as(h2c.P_f64), k, float(kappa), float(diagonal),
                                             orders.ctypes.data_as(C.POINTER(C.c_int32)), float(eps_recompress),
                                             int(threads))
    return _take_h2(h, tree, structure)


def build_fd_laplacian(tree: ClusterTree, structure: BlockTree, points: np.ndarray, h: float) -> H2Matrix:
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    hd = h2c.lib().h2c_build_fd_laplacian(C.byref(tree.desc()), C.byref(structure.desc()),
                                          pts.ctypes.data_as(h2c.P_f64), float(h))
    return _take_h2(hd, tree, structure)


# ---------------------------------------------------------------------------
def svd_truncate_gram(gram: np.ndarray, eps: float, ctx: Optional[Context] = None):
    """svd_truncate_gram (truncation.cpp:9-47) on the B200 -> (basis, degenerate)."""
    g = np.asfortranarray(gram)
    if g.ndim != 2 or g.shape[0] != g.shape[1] or g.shape[0] < 1:
        raise ConfigError("svd_truncate_gram: gram matrix must be square and non-empty")
    cplx = np.iscomplexobj(g)
    g = np.asfortranarray(g, dtype=np.complex128 if cplx else np.float64)
    ctx = ctx or default_context()
    n = g.shape[0]
    basis = np.zeros((n, n), dtype=g.dtype, order="F")
    rank, degen = C.c_int(), C.c_int()
    rc = h2c.lib().h2c_truncate_gram(ctx.handle, int(cplx), g.ctypes.data_as(h2c.P_f64), n, float(eps),
                                     basis.ctypes.data_as(h2c.P_f64), C.byref(rank), C.byref(degen))
    raise_for(rc, h2c.last_error(ctx.handle))
    return basis[:, :rank.value].copy(), bool(degen.value)


def random_vector(n: int, seed: int, complex_: bool = False) -> np.ndarray:
    """random_vector (metrics.cpp:11-35)."""
    out = np.zeros(n, dtype=np.complex128 if complex_ else np.float64)
    raise_for(h2c.lib().h2c_random_vector(int(n), int(seed), int(complex_), out.ctypes.data_as(h2c.P_f64)),
              h2c.last_error())
    return out


def mvp(a: H2Matrix, x: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
    """Exact H^2 MVP on the B200 (h2_matrix.cpp:213-278); x is [N] or [N, nv]."""
    ctx = ctx or default_context()
    xx = np.asfortranarray(x, dtype=a.dtype)
    nv = 1 if xx.ndim == 1 else xx.shape[1]
    y = np.zeros_like(xx, order="F")
    rc = h2c.lib().h2c_mvp(ctx.handle, C.byref(a.desc()), xx.ctypes.data_as(h2c.P_f64), nv,
                           y.ctypes.data_as(h2c.P_f64))
    raise_for(rc, h2c.last_error(ctx.handle))
    return y


def h2_to_dense(a: H2Matrix, ctx: Optional[Context] = None) -> np.ndarray:
    """Dense N x N materialisation on the B200 (h2_matrix.cpp:124-137), original point ordering."""
    ctx = ctx or default_context()
    n = a.size()
    out = np.zeros((n, n), dtype=a.dtype, order="F")
    rc = h2c.lib().h2c_to_dense(ctx.handle, C.byref(a.desc()), out.ctypes.data_as(h2c.P_f64))
    raise_for(rc, h2c.last_error(ctx.handle))
    return out


def relative_error(a: H2Matrix, b: H2Matrix, c: H2Matrix, seed: int, ctx: Optional[Context] = None) -> float:
    """||C x - A (B x)|| / ||A (B x)|| with x = random_vector(seed) (metrics.cpp:37-55), on the B200."""
    if not (a.tree is b.tree is c.tree):
        raise ConfigError("relative_error: operands must share the cluster tree")
    x = random_vector(a.size(), seed, a.scalar == h2c.H2C_COMPLEX)
    ref = mvp(a, mvp(b, x, ctx), ctx)
    cx = mvp(c, x, ctx)
    rn = np.linalg.norm(ref)
    return float(np.linalg.norm(cx)) if rn == 0 else float(np.linalg.norm(cx - ref) / rn)


def plan_stats(structure: BlockTree) -> list[dict]:
    """Per-level sizes of the structure plan (blocks, targets, triples)."""
    cap = structure.depth + 1
    out = np.zeros(10 * cap, dtype=np.int64)
    n = h2c.lib().h2c_plan_stats(C.byref(structure.tree.desc()), C.byref(structure.desc()),
                                 out.ctypes.data_as(h2c.P_i64), cap)
    if n < 0:
        raise h2c.InvariantError(h2c.last_error())
    keys = ["clusters", "admissible", "near", "pending", "nonleaf", "merged", "RxR", "FRxR", "RxF", "FxF"]
    return [dict(level=l, **{k: int(out[10 * l + i]) for i, k in enumerate(keys)}) for l in range(n)]


class _ResultOwner:
    """Keeps the library-owned result (pinned host values) alive while a view exists."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                h2c.lib().h2c_result_free(self.handle)
                self.handle = None
        except Exception:
            pass


def _result(handle, a: H2Matrix) -> MmpResult:
    """Wraps an h2c_result: the value array is a zero-copy view of the library's pinned buffer."""
    L = h2c.lib()
    owner = _ResultOwner(handle)
    d = h2c_matrix()
    L.h2c_result_matrix(handle, C.byref(d))
    nc, nb = a.tree.n_clusters, a.structure.n_blocks
    w = 2 if d.scalar == h2c.H2C_COMPLEX else 1
    n = w * d.n_values
    if n:
        # the array's base chain ends in a ctypes buffer that holds the owner, so any view of
        # the values (even without the H2Matrix) keeps the library's pinned buffer alive
        buf = (C.c_double * n).from_address(C.cast(d.values, C.c_void_p).value)
        buf._owner = owner
        vals = np.frombuffer(buf, dtype=np.float64)
    else:
        vals = np.zeros(0)
    if w == 2:
        vals = vals.view(np.complex128)
    prod = H2Matrix(a.tree, a.structure, d.scalar, h2c._copy(d.row_rank, nc, np.int32),
                    h2c._copy(d.col_rank, nc, np.int32), h2c._copy(d.row_degenerate, nc, np.uint8),
                    h2c._copy(d.col_degenerate, nc, np.uint8), h2c._copy(d.row_offset, nc, np.int64),
                    h2c._copy(d.col_offset, nc, np.int64), h2c._copy(d.block_offset, nb, np.int64), vals)
    prod._owner = owner
    r = h2c_report()
    L.h2c_result_report(handle, C.byref(r))
    return MmpResult(prod, MmpReport.from_desc(r))


def mmp(a: H2Matrix, b: H2Matrix, eps_trunc: float, ctx: Optional[Context] = None) -> MmpResult:
    """Accuracy-controlled product C = A*B (mmp.cpp:688-691) on the B200."""
    ctx = ctx or default_context()
    out = C.c_void_p()
    rc = h2c.lib().h2c_mmp(ctx.handle, C.byref(a.desc()), C.byref(b.desc()), float(eps_trunc), C.byref(out))
    raise_for(rc, h2c.last_error(ctx.handle))
    return _result(out, a)


def formatted_mmp(a: H2Matrix, b: H2Matrix, ctx: Optional[Context] = None) -> MmpResult:
    """Baseline formatted product with unchanged bases (mmp.cpp:716-719)."""
    ctx = ctx or default_context()
    out = C.c_void_p()
    rc = h2c.lib().h2c_formatted_mmp(ctx.handle, C.byref(a.desc()), C.byref(b.desc()), C.byref(out))
    raise_for(rc, h2c.last_error(ctx.handle))
    return _result(out, a)


def count_report(a: H2Matrix, b: H2Matrix, c: H2Matrix, adaptive: bool = True, eps_trunc: float = 0.0) -> MmpReport:
    """Host-side MmpReport counters of C = A*B from structure and ranks (h2c_count_report)."""
    out = C.c_void_p()
    rc = h2c.lib().h2c_count_report(C.byref(a.desc()), C.byref(b.desc()), C.byref(c.desc()), int(adaptive),
                                    float(eps_trunc), C.byref(out))
    raise_for(rc, h2c.last_error())
    try:
        r = h2c_report()
        h2c.lib().h2c_result_report(out, C.byref(r))
        return MmpReport.from_desc(r)
    finally:
        h2c.lib().h2c_result_free(out)


class ResidentOperand:
    """An operand uploaded once to HBM (h2c_upload) for repeated products."""

    def __init__(self, m: H2Matrix, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.matrix = m
        h = C.c_void_p()
        rc = h2c.lib().h2c_upload(self.ctx.handle, C.byref(m.desc()), C.byref(h))
        raise_for(rc, h2c.last_error(self.ctx.handle))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                h2c.lib().h2c_operand_free(self._h)
        except Exception:
            pass


def mmp_resident(a: ResidentOperand, b: ResidentOperand, eps_trunc: float, adaptive: bool = True,
                 want_report: bool = False):
    """Runs the product on resident operands; returns (device_seconds, report|None)."""
    ctx = a.ctx
    secs = C.c_double()
    out = C.c_void_p() if want_report else None
    rc = h2c.lib().h2c_mmp_resident(ctx.handle, a._h, b._h, float(eps_trunc), int(adaptive), C.byref(secs),
                                    C.byref(out) if want_report else None)
    raise_for(rc, h2c.last_error(ctx.handle))
    rep = None
    if want_report:
        r = h2c_report()
        h2c.lib().h2c_result_report(out, C.byref(r))
        rep = MmpReport.from_desc(r)
        h2c.lib().h2c_result_free(out)
    return secs.value, rep


class PinnedArray:
    """numpy view over pinned host memory (h2c_host_alloc)."""

    def __init__(self, n: int, dtype=np.float64):
        self.nbytes = max(1, int(n) * np.dtype(dtype).itemsize)
        self._p = h2c.lib().h2c_host_alloc(self.nbytes)
        if not self._p:
            raise MemoryError(h2c.last_error())
        buf = (C.c_char * self.nbytes).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(n))

    def __del__(self):
        try:
            if self._p:
                h2c.lib().h2c_host_free(self._p)
                self._p = None
        except Exception:
            pass


def pin_matrix(m: H2Matrix) -> tuple[H2Matrix, PinnedArray]:
    """Copy of `m` whose value array lives in pinned host memory."""
    pa = PinnedArray(len(m.values), m.values.dtype)
    pa.array[:] = m.values
    return m.copy_with(pa.array), pa
