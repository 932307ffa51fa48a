"""ctypes layer over libh2mmp_b200.so and the Python mirror of the reference's
H^2 data model (proj/core/include/h2mmp/{cluster_tree,block_tree,h2_matrix,
mmp}.hpp).

The descriptors below are byte-for-byte the structs of include/h2c_types.h.
Python objects own numpy arrays; a descriptor is built once per object and
cached, so two matrices that share the same ClusterTree / BlockTree objects
pass the same descriptor ADDRESSES to the library - the shared_ptr identity
check of the reference (mmp.cpp:59) becomes an address check.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

PKG = Path(__file__).resolve().parent
LIBPATH = PKG / "lib" / "libh2mmp_b200.so"

H2C_REAL, H2C_COMPLEX = 0, 1
ADMISSIBLE, INADMISSIBLE_LEAF, SUBDIVIDED = 0, 1, 2
H2C_OK, H2C_ERR_CONFIG, H2C_ERR_INVARIANT, H2C_ERR_CUDA, H2C_ERR_ALLOC = 0, 2, 3, 4, 5


class ConfigError(ValueError):
    """h2mmp::ConfigError (errors.hpp:9-13)."""


class InvariantError(RuntimeError):
    """h2mmp::InvariantError (errors.hpp:21-25)."""


class DeviceError(RuntimeError):
    """CUDA failure inside the library (no CPU fallback exists)."""


def raise_for(code: int, msg: str) -> None:
    if code == H2C_OK:
        return
    if code == H2C_ERR_CONFIG:
        raise ConfigError(msg)
    if code == H2C_ERR_INVARIANT:
        raise InvariantError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------------------
# descriptors (include/h2c_types.h)
P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_u8 = C.POINTER(C.c_uint8)
P_f64 = C.POINTER(C.c_double)


class h2c_tree(C.Structure):
    _fields_ = [("n_points", C.c_int32), ("depth", C.c_int32), ("leafsize", C.c_int32),
                ("n_clusters", C.c_int32), ("parent", P_i32), ("child0", P_i32), ("child1", P_i32),
                ("level", P_i32), ("begin", P_i32), ("end", P_i32), ("bbox", P_f64), ("perm", P_i32)]


class h2c_blocks(C.Structure):
    _fields_ = [("depth", C.c_int32), ("c_sp", C.c_int32), ("eta", C.c_double), ("n_blocks", C.c_int64),
                ("level_ptr", P_i64), ("row", P_i32), ("col", P_i32), ("kind", P_u8)]


class h2c_matrix(C.Structure):
    _fields_ = [("tree", C.POINTER(h2c_tree)), ("blocks", C.POINTER(h2c_blocks)), ("scalar", C.c_int32),
                ("row_rank", P_i32), ("col_rank", P_i32), ("row_degenerate", P_u8), ("col_degenerate", P_u8),
                ("row_offset", P_i64), ("col_offset", P_i64), ("block_offset", P_i64), ("values", P_f64),
                ("n_values", C.c_int64)]


class h2c_report(C.Structure):
    _fields_ = [("eps_trunc", C.c_double), ("adaptive", C.c_int32), ("n_levels", C.c_int32),
                ("flops", C.c_int64), ("case_flops", C.c_int64 * 4), ("wall_seconds", C.c_double),
                ("pending_after_split", C.c_int32), ("max_row_rank", P_i64), ("max_col_rank", P_i64),
                ("case_products", P_i64), ("max_case1_terms", P_i32), ("max_case2_terms", P_i32),
                ("max_case3_terms", P_i32), ("flops_exec", C.c_int64), ("device_seconds", C.c_double),
                ("plan_seconds", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _copy(p, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dtype, copy=True)


# ---------------------------------------------------------------------------
# Python model
class ClusterTree:
    """ClusterTree (cluster_tree.hpp:31-41): flat arrays indexed by cluster id."""

    def __init__(self, n_points, depth, leafsize, parent, child0, child1, level, begin, end, bbox, perm):
        self.n_points = int(n_points)
        self.depth = int(depth)
        self.leafsize = int(leafsize)
        self.parent = np.ascontiguousarray(parent, dtype=np.int32)
        self.child0 = np.ascontiguousarray(child0, dtype=np.int32)
        self.child1 = np.ascontiguousarray(child1, dtype=np.int32)
        self.level = np.ascontiguousarray(level, dtype=np.int32)
        self.begin = np.ascontiguousarray(begin, dtype=np.int32)
        self.end = np.ascontiguousarray(end, dtype=np.int32)
        self.bbox = np.ascontiguousarray(bbox, dtype=np.float64).reshape(-1, 6)
        self.perm = np.ascontiguousarray(perm, dtype=np.int32)
        self.inv_perm = np.empty_like(self.perm)
        self.inv_perm[self.perm] = np.arange(self.n_points, dtype=np.int32)
        self._desc: Optional[h2c_tree] = None
        self.points: Optional[np.ndarray] = None

    @property
    def n_clusters(self) -> int:
        return len(self.parent)

    def size(self, c: int) -> int:
        return int(self.end[c] - self.begin[c])

    def is_leaf(self, c: int) -> bool:
        return self.child0[c] < 0

    @property
    def levels(self) -> list[np.ndarray]:
        out = []
        for l in range(self.depth + 1):
            ids = np.nonzero(self.level == l)[0]
            out.append(ids[np.argsort(self.begin[ids], kind="stable")].astype(np.int32))
        return out

    def desc(self) -> h2c_tree:
        if self._desc is None:
            self._desc = h2c_tree(self.n_points, self.depth, self.leafsize, self.n_clusters,
                                  _ptr(self.parent, P_i32), _ptr(self.child0, P_i32), _ptr(self.child1, P_i32),
                                  _ptr(self.level, P_i32), _ptr(self.begin, P_i32), _ptr(self.end, P_i32),
                                  _ptr(self.bbox, P_f64), _ptr(self.perm, P_i32))
        return self._desc

    @staticmethod
    def from_desc(d: h2c_tree) -> "ClusterTree":
        n = d.n_clusters
        return ClusterTree(d.n_points, d.depth, d.leafsize, _copy(d.parent, n, np.int32), _copy(d.child0, n, np.int32),
                           _copy(d.child1, n, np.int32), _copy(d.level, n, np.int32), _copy(d.begin, n, np.int32),
                           _copy(d.end, n, np.int32),
                           _copy(d.bbox, 6 * n, np.float64) if d.bbox else np.zeros(6 * n),
                           _copy(d.perm, d.n_points, np.int32))

    def same_as(self, o: "ClusterTree") -> bool:
        return (self.depth == o.depth and self.n_points == o.n_points and
                all(np.array_equal(getattr(self, f), getattr(o, f))
                    for f in ("parent", "child0", "child1", "level", "begin", "end", "perm", "bbox")))


class BlockTree:
    """BlockTree (block_tree.hpp:40-73) over one shared cluster tree."""

    def __init__(self, tree: ClusterTree, eta, c_sp, level_ptr, row, col, kind):
        self.tree = tree
        self.eta = float(eta)
        self.c_sp = int(c_sp)
        self.level_ptr = np.ascontiguousarray(level_ptr, dtype=np.int64)
        self.row = np.ascontiguousarray(row, dtype=np.int32)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.kind = np.ascontiguousarray(kind, dtype=np.uint8)
        self._desc: Optional[h2c_blocks] = None
        self._index = None

    @property
    def depth(self) -> int:
        return self.tree.depth

    @property
    def n_blocks(self) -> int:
        return len(self.row)

    def rows(self) -> ClusterTree:
        return self.tree

    def cols(self) -> ClusterTree:
        return self.tree

    def level_blocks(self, l: int):
        a, b = self.level_ptr[l], self.level_ptr[l + 1]
        return [((int(self.row[i]), int(self.col[i])), int(self.kind[i])) for i in range(a, b)]

    def index(self) -> dict:
        if self._index is None:
            self._index = {(int(r), int(c)): i for i, (r, c) in enumerate(zip(self.row, self.col))}
        return self._index

    def kind_of(self, t: int, s: int) -> Optional[int]:
        i = self.index().get((t, s))
        return None if i is None else int(self.kind[i])

    def admissible_count(self) -> int:
        return int(np.sum(self.kind == ADMISSIBLE))

    def inadmissible_count(self) -> int:
        return int(np.sum(self.kind == INADMISSIBLE_LEAF))

    def desc(self) -> h2c_blocks:
        if self._desc is None:
            self._desc = h2c_blocks(self.depth, self.c_sp, self.eta, self.n_blocks, _ptr(self.level_ptr, P_i64),
                                    _ptr(self.row, P_i32), _ptr(self.col, P_i32), _ptr(self.kind, P_u8))
        return self._desc

    @staticmethod
    def from_desc(tree: ClusterTree, d: h2c_blocks) -> "BlockTree":
        n = d.n_blocks
        return BlockTree(tree, d.eta, d.c_sp, _copy(d.level_ptr, d.depth + 2, np.int64), _copy(d.row, n, np.int32),
                         _copy(d.col, n, np.int32), _copy(d.kind, n, np.uint8))


class H2Matrix:
    """H2Matrix<Scalar> (h2_matrix.hpp:38-48) in the flat layout of h2c_types.h."""

    def __init__(self, tree: ClusterTree, structure: BlockTree, scalar: int, row_rank, col_rank, row_degenerate,
                 col_degenerate, row_offset, col_offset, block_offset, values: np.ndarray):
        if structure.tree is not tree:
            raise ConfigError("H2Matrix: structure must be built over the given tree")
        self.tree = tree
        self.structure = structure
        self.scalar = int(scalar)
        self.row_rank = np.ascontiguousarray(row_rank, dtype=np.int32)
        self.col_rank = np.ascontiguousarray(col_rank, dtype=np.int32)
        self.row_degenerate = np.ascontiguousarray(row_degenerate, dtype=np.uint8)
        self.col_degenerate = np.ascontiguousarray(col_degenerate, dtype=np.uint8)
        self.row_offset = np.ascontiguousarray(row_offset, dtype=np.int64)
        self.col_offset = np.ascontiguousarray(col_offset, dtype=np.int64)
        self.block_offset = np.ascontiguousarray(block_offset, dtype=np.int64)
        dt = np.complex128 if self.scalar == H2C_COMPLEX else np.float64
        self.values = values if (values.dtype == dt and values.flags.c_contiguous) else np.ascontiguousarray(values, dtype=dt)
        self._desc = None

    @property
    def dtype(self):
        return np.complex128 if self.scalar == H2C_COMPLEX else np.float64

    def size(self) -> int:
        return self.tree.n_points

    def desc(self) -> h2c_matrix:
        if self._desc is None:
            self._desc = h2c_matrix(C.pointer(self.tree.desc()), C.pointer(self.structure.desc()), self.scalar,
                                    _ptr(self.row_rank, P_i32), _ptr(self.col_rank, P_i32),
                                    _ptr(self.row_degenerate, P_u8), _ptr(self.col_degenerate, P_u8),
                                    _ptr(self.row_offset, P_i64), _ptr(self.col_offset, P_i64),
                                    _ptr(self.block_offset, P_i64), self.values.ctypes.data_as(P_f64),
                                    len(self.values))
        return self._desc

    # views (column-major blocks of the flat value array)
    def _view(self, off: int, r: int, c: int) -> np.ndarray:
        if r * c == 0:
            return np.zeros((r, c), dtype=self.dtype)
        return self.values[off:off + r * c].reshape(c, r).T

    def row_basis(self, c: int) -> np.ndarray:
        t = self.tree
        r = t.size(c) if t.is_leaf(c) else int(self.row_rank[t.child0[c]] + self.row_rank[t.child1[c]])
        return self._view(int(self.row_offset[c]), r, int(self.row_rank[c])) if self.row_offset[c] >= 0 \
            else np.zeros((0, 0), self.dtype)

    def col_basis(self, c: int) -> np.ndarray:
        t = self.tree
        r = t.size(c) if t.is_leaf(c) else int(self.col_rank[t.child0[c]] + self.col_rank[t.child1[c]])
        return self._view(int(self.col_offset[c]), r, int(self.col_rank[c])) if self.col_offset[c] >= 0 \
            else np.zeros((0, 0), self.dtype)

    def block(self, b: int) -> np.ndarray:
        s, t = self.structure, self.tree
        r, c = int(s.row[b]), int(s.col[b])
        if s.kind[b] == ADMISSIBLE:
            return self._view(int(self.block_offset[b]), int(self.row_rank[r]), int(self.col_rank[c]))
        if s.kind[b] == INADMISSIBLE_LEAF:
            return self._view(int(self.block_offset[b]), t.size(r), t.size(c))
        raise KeyError("subdivided blocks store nothing")

    def coupling(self, t: int, s: int) -> np.ndarray:
        return self.block(self.structure.index()[(t, s)])

    def full(self, t: int, s: int) -> np.ndarray:
        return self.block(self.structure.index()[(t, s)])

    def copy_with(self, values: np.ndarray) -> "H2Matrix":
        return H2Matrix(self.tree, self.structure, self.scalar, self.row_rank, self.col_rank, self.row_degenerate,
                        self.col_degenerate, self.row_offset, self.col_offset, self.block_offset, values)

    @staticmethod
    def from_desc(tree: ClusterTree, structure: BlockTree, d: h2c_matrix) -> "H2Matrix":
        nc, nb = tree.n_clusters, structure.n_blocks
        w = 2 if d.scalar == H2C_COMPLEX else 1
        vals = _copy(d.values, w * d.n_values, np.float64)
        if w == 2:
            vals = vals.view(np.complex128)
        return H2Matrix(tree, structure, d.scalar, _copy(d.row_rank, nc, np.int32), _copy(d.col_rank, nc, np.int32),
                        _copy(d.row_degenerate, nc, np.uint8), _copy(d.col_degenerate, nc, np.uint8),
                        _copy(d.row_offset, nc, np.int64), _copy(d.col_offset, nc, np.int64),
                        _copy(d.block_offset, nb, np.int64), vals)


@dataclass
class LevelStats:
    """LevelStats (mmp.hpp:16-24)."""
    level: int = 0
    max_row_rank: int = 0
    max_col_rank: int = 0
    case_products: list = field(default_factory=lambda: [0, 0, 0, 0])
    max_case1_terms: int = 0
    max_case2_terms: int = 0
    max_case3_terms: int = 0


@dataclass
class MmpReport:
    """MmpReport (mmp.hpp:26-42) + B200 extensions."""
    eps_trunc: float = 0.0
    adaptive: bool = True
    levels: list = field(default_factory=list)
    flops: int = 0
    case_flops: list = field(default_factory=lambda: [0, 0, 0, 0])
    wall_seconds: float = 0.0
    pending_after_split: int = 0
    flops_exec: int = 0
    device_seconds: float = 0.0
    plan_seconds: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def max_rank(self) -> int:
        return max([0] + [max(s.max_row_rank, s.max_col_rank) for s in self.levels])

    @staticmethod
    def from_desc(r: h2c_report) -> "MmpReport":
        n = r.n_levels
        lv = []
        for l in range(n):
            lv.append(LevelStats(l, int(r.max_row_rank[l]), int(r.max_col_rank[l]),
                                 [int(r.case_products[4 * l + c]) for c in range(4)], int(r.max_case1_terms[l]),
                                 int(r.max_case2_terms[l]), int(r.max_case3_terms[l])))
        return MmpReport(r.eps_trunc, bool(r.adaptive), lv, int(r.flops), [int(x) for x in r.case_flops],
                         r.wall_seconds, r.pending_after_split, int(r.flops_exec), r.device_seconds, r.plan_seconds,
                         int(r.h2d_bytes), int(r.d2h_bytes))


@dataclass
class MmpResult:
    """MmpResult<Scalar> (mmp.hpp:44-48)."""
    product: H2Matrix
    report: MmpReport


# ---------------------------------------------------------------------------
_lib = None


# CPU-only input generator (structure + synthetic operands, no MMP entry points):
# oracle/_build/libh2inputs.so, built from this package's host sources
INPUTS_LIBPATH = PKG.parent / "oracle" / "_build" / "libh2inputs.so"
_lib_path = LIBPATH


def use_inputs_library() -> None:
    """Bind the host-only input generator instead of the B200 library (bench.py's
    reference arm builds its operands without mapping libh2mmp_b200.so).  Must be
    called before the first lib(); the MMP entry points are then unavailable."""
    global _lib_path
    if _lib is not None and _lib_path != INPUTS_LIBPATH:
        raise RuntimeError("the B200 library is already loaded")
    _lib_path = INPUTS_LIBPATH


def _sig(L, name: str, attr: str, value) -> None:
    f = getattr(L, name, None)
    if f is None:
        if _lib_path == INPUTS_LIBPATH:
            return  # not part of the input generator
        raise ImportError(f"{name} missing from {_lib_path}")
    setattr(f, attr, value)


def lib() -> C.CDLL:
    """The B200 library; raises if it is missing (there is no fallback)."""
    global _lib
    if _lib is None:
        path = _lib_path
        if not path.exists():
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(str(path))
        _sig(L, "h2c_version", "restype", C.c_int)
        _sig(L, "h2c_last_error", "restype", C.c_char_p)
        _sig(L, "h2c_last_error", "argtypes", [C.c_void_p])
        _sig(L, "h2c_create", "restype", C.c_void_p)
        _sig(L, "h2c_create", "argtypes", [C.c_int])
        _sig(L, "h2c_destroy", "argtypes", [C.c_void_p])
        _sig(L, "h2c_kernel_launches", "restype", C.c_int64)
        _sig(L, "h2c_kernel_launches", "argtypes", [C.c_void_p])
        _sig(L, "h2c_stream", "restype", C.c_void_p)
        _sig(L, "h2c_stream", "argtypes", [C.c_void_p])
        _sig(L, "h2c_set_profile", "argtypes", [C.c_void_p, C.c_int])
        _sig(L, "h2c_profile_count", "restype", C.c_int)
        _sig(L, "h2c_profile_count", "argtypes", [C.c_void_p])
        _sig(L, "h2c_profile_get", "restype", C.c_int)
        _sig(L, "h2c_profile_bytes", "restype", C.c_int64)
        _sig(L, "h2c_profile_bytes", "argtypes", [C.c_void_p, C.c_int])
        _sig(L, "h2c_profile_get", "argtypes", [C.c_void_p, C.c_int, C.c_char_p, C.c_int, P_i64, C.POINTER(C.c_double), P_i64])
        _sig(L, "h2c_build_structure", "restype", C.c_void_p)
        _sig(L, "h2c_build_structure", "argtypes", [P_f64, C.c_int, C.c_int, C.c_double])
        _sig(L, "h2c_structure_tree", "argtypes", [C.c_void_p, C.POINTER(h2c_tree)])
        _sig(L, "h2c_structure_blocks", "argtypes", [C.c_void_p, C.POINTER(h2c_blocks)])
        _sig(L, "h2c_structure_free", "argtypes", [C.c_void_p])
        _sig(L, "h2c_target_status", "restype", C.c_int)
        _sig(L, "h2c_target_status", "argtypes", [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), C.c_int, C.c_int])
        _sig(L, "h2c_random_cloud", "restype", C.c_int)
        _sig(L, "h2c_random_cloud", "argtypes", [C.c_int, C.c_uint64, P_f64])
        _sig(L, "h2c_build_chebyshev", "restype", C.c_void_p)
        _sig(L, "h2c_build_chebyshev", "argtypes", [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), P_f64, C.c_int, C.c_double,
                                          C.c_double, C.c_int, C.c_double, C.c_int])
        _sig(L, "h2c_build_chebyshev_orders", "restype", C.c_void_p)
        _sig(L, "h2c_build_chebyshev_orders", "argtypes", [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), P_f64, C.c_int,
                                                 C.c_double, C.c_double, C.POINTER(C.c_int32), C.c_double, C.c_int])
        _sig(L, "h2c_build_fd_laplacian", "restype", C.c_void_p)
        _sig(L, "h2c_build_fd_laplacian", "argtypes", [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), P_f64, C.c_double])
        _sig(L, "h2c_h2_desc", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix)])
        _sig(L, "h2c_h2_free", "argtypes", [C.c_void_p])
        _sig(L, "h2c_mmp", "restype", C.c_int)
        _sig(L, "h2c_mmp", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix), C.POINTER(h2c_matrix), C.c_double,
                                       C.POINTER(C.c_void_p)])
        _sig(L, "h2c_formatted_mmp", "restype", C.c_int)
        _sig(L, "h2c_formatted_mmp", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix), C.POINTER(h2c_matrix),
                                        C.POINTER(C.c_void_p)])
        _sig(L, "h2c_result_matrix", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix)])
        _sig(L, "h2c_result_report", "argtypes", [C.c_void_p, C.POINTER(h2c_report)])
        _sig(L, "h2c_result_free", "argtypes", [C.c_void_p])
        _sig(L, "h2c_upload", "restype", C.c_int)
        _sig(L, "h2c_upload", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix), C.POINTER(C.c_void_p)])
        _sig(L, "h2c_operand_free", "argtypes", [C.c_void_p])
        _sig(L, "h2c_mmp_resident", "restype", C.c_int)
        _sig(L, "h2c_mmp_resident", "argtypes", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_void_p)])
        _sig(L, "h2c_count_report", "restype", C.c_int)
        _sig(L, "h2c_count_report", "argtypes", [C.POINTER(h2c_matrix)] * 3 + [C.c_int, C.c_double, C.POINTER(C.c_void_p)])
        _sig(L, "h2c_mvp", "restype", C.c_int)
        _sig(L, "h2c_mvp", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix), P_f64, C.c_int, P_f64])
        _sig(L, "h2c_to_dense", "restype", C.c_int)
        _sig(L, "h2c_to_dense", "argtypes", [C.c_void_p, C.POINTER(h2c_matrix), P_f64])
        _sig(L, "h2c_mvp_resident", "restype", C.c_int)
        _sig(L, "h2c_mvp_resident", "argtypes", [C.c_void_p, C.c_void_p, P_f64, C.c_int, P_f64])
        _sig(L, "h2c_random_vector", "restype", C.c_int)
        _sig(L, "h2c_random_vector", "argtypes", [C.c_int, C.c_uint64, C.c_int, P_f64])
        _sig(L, "h2c_truncate_gram", "restype", C.c_int)
        _sig(L, "h2c_truncate_gram", "argtypes", [C.c_void_p, C.c_int, P_f64, C.c_int, C.c_double, P_f64, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)])
        _sig(L, "h2c_plan_stats", "restype", C.c_int)
        _sig(L, "h2c_plan_stats", "argtypes", [C.POINTER(h2c_tree), C.POINTER(h2c_blocks), P_i64, C.c_int])
        _sig(L, "h2c_host_alloc", "restype", C.c_void_p)
        _sig(L, "h2c_host_alloc", "argtypes", [C.c_size_t])
        _sig(L, "h2c_host_free", "argtypes", [C.c_void_p])
        _lib = L
    return _lib


def last_error(ctx=None) -> str:
    m = lib().h2c_last_error(ctx)
    return m.decode() if m else ""


# exported symbols declared in include/h2c.h (checked by the CPU test suite)
def declared_symbols(header: Path = PKG.parent / "include" / "h2c.h") -> list[str]:
    import re
    text = header.read_text()
    return sorted(set(re.findall(r"\b(h2c_[a-z0-9_]+)\s*\(", text)))
