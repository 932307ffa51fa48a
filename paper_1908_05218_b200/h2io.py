"""Binary flat H^2 serialisation ("h2bin/1").

The reference stores matrices as JSON ("h2json/1", proj/core/src/h2_io.cpp:14-319),
which is impractical for multi-GB operands.  h2bin/1 stores exactly the flat
layout of include/h2c_types.h (one numpy .npz: tree, blocks, ranks, offsets,
values) and round-trips bit-exactly, with the reference's failure behaviour of
raising LoadError on malformed or truncated input (h2_io.hpp:15-31).
"""
from __future__ import annotations

import zipfile

import numpy as np

from .h2c import BlockTree, ClusterTree, H2Matrix

FORMAT = "h2bin/1"


class LoadError(RuntimeError):
    """h2mmp::LoadError (errors.hpp:27-29)."""


def save_h2(path: str, m: H2Matrix) -> None:
    t, s = m.tree, m.structure
    np.savez(path, format=np.array(FORMAT), n_points=t.n_points, depth=t.depth, leafsize=t.leafsize,
             parent=t.parent, child0=t.child0, child1=t.child1, level=t.level, begin=t.begin, end=t.end,
             bbox=t.bbox, perm=t.perm, eta=s.eta, c_sp=s.c_sp, level_ptr=s.level_ptr, row=s.row, col=s.col,
             kind=s.kind, scalar=m.scalar, row_rank=m.row_rank, col_rank=m.col_rank,
             row_degenerate=m.row_degenerate, col_degenerate=m.col_degenerate, row_offset=m.row_offset,
             col_offset=m.col_offset, block_offset=m.block_offset, values=m.values)


def load_h2(path: str, tree: ClusterTree | None = None, structure: BlockTree | None = None) -> H2Matrix:
    """Loads a matrix; pass an existing tree/structure to share them (required for mmp operands)."""
    try:
        with np.load(path, allow_pickle=False) as z:
            if str(z["format"]) != FORMAT:
                raise LoadError(f"{path}: not an {FORMAT} file")
            d = {k: z[k] for k in z.files}
    except LoadError:
        raise
    except (OSError, ValueError, KeyError, EOFError, zipfile.BadZipFile) as e:
        raise LoadError(f"{path}: malformed or truncated {FORMAT} file ({e})") from e
    t = ClusterTree(d["n_points"], d["depth"], d["leafsize"], d["parent"], d["child0"], d["child1"], d["level"],
                    d["begin"], d["end"], d["bbox"], d["perm"])
    if tree is not None:
        if not tree.same_as(t):
            raise LoadError(f"{path}: cluster tree differs from the one supplied")
        t = tree
    s = BlockTree(t, d["eta"], d["c_sp"], d["level_ptr"], d["row"], d["col"], d["kind"])
    if structure is not None:
        if structure.tree is not t or not all(np.array_equal(getattr(structure, f), d[f])
                                               for f in ("level_ptr", "row", "col", "kind")):
            raise LoadError(f"{path}: block structure differs from the one supplied")
        s = structure
    nv = len(d["values"])
    for off in (d["row_offset"], d["col_offset"], d["block_offset"]):
        if len(off) and off.max() > nv:
            raise LoadError(f"{path}: offset past the value array")
    return H2Matrix(t, s, int(d["scalar"]), d["row_rank"], d["col_rank"], d["row_degenerate"], d["col_degenerate"],
                    d["row_offset"], d["col_offset"], d["block_offset"], d["values"])
