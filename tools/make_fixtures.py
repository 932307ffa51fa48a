#!/usr/bin/env python3
"""Compact full-size oracle fixtures for the default `-m gpu` suite (tests/golden/full_<cfg>.npz).

Run on the GPU box (its host cores run the all-cores oracle; the operands are built with the
package's constructors exactly as tests/test_full_size_fixtures.py builds them):

    python tools/make_fixtures.py cfg2 cfg3 cfg5s

Per BASELINE configuration at its full size it stores what the parity bar of BASELINE.json
needs, without the multi-GB product itself:
  * C_ref's per-cluster ranks and degenerate flags, every MmpReport counter, and the oracle's
    smallest eigenvalue-to-threshold margin (rank flips are only allowed below 1e-10);
  * a two-sided random sketch S = W^H (C_ref X) of the product, with X, W 16 seeded
    `random_vector`s each (metrics.cpp:17-35; seeds 1000+s and 2000+s): ||W^H (C - C_ref) X||_F /
    ||S||_F estimates ||C - C_ref||_F / ||C_ref||_F;
  * C_ref X exactly at 1024 seeded rows (all 16 columns) and the column norms of C_ref X;
  * the same sketch of the operands (W^H A X, W^H B X): a changed constructor makes the test fail
    as "fixture stale" instead of comparing different products.
C_ref X uses the oracle's exact H^2 MVP (h2_matrix.cpp:213-278).  The fixture is test data only.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NPROBE = 16
NROWS = 1024


def probe_vectors(n: int, cplx: bool):
    from oracle import pyoracle as O
    X = np.stack([O.random_vector(n, 1000 + s, cplx) for s in range(NPROBE)], 1)
    Wv = np.stack([O.random_vector(n, 2000 + s, cplx) for s in range(NPROBE)], 1)
    return np.asfortranarray(X), np.asfortranarray(Wv)


def probe_rows(n: int) -> np.ndarray:
    return np.sort(np.random.default_rng(12345).choice(n, size=min(NROWS, n), replace=False))


def make(name: str, threads: int) -> dict:
    import bench
    import paper_1908_05218_b200 as P
    from oracle import pyoracle as O
    W = bench.build_workload(name)
    A, B, eps = W["A"], W["B"], W["eps"]
    cplx = A.scalar == P.H2C_COMPLEX
    n = W["n"]
    t0 = time.perf_counter()
    ref, margin = O.mmp(A, B, eps, with_margin=True, threads=threads)
    t_oracle = time.perf_counter() - t0
    X, Wv = probe_vectors(n, cplx)
    t0 = time.perf_counter()
    Y = O.mvp_multi(ref.product, X, threads)
    SA = Wv.conj().T @ O.mvp_multi(A, X, threads)
    SB = SA if B is A else Wv.conj().T @ O.mvp_multi(B, X, threads)
    t_probe = time.perf_counter() - t0
    rows = probe_rows(n)
    rep = ref.report
    lv = rep.levels
    out = dict(
        name=name, N=n, eps=eps, margin=margin, threads=threads, oracle_seconds=t_oracle,
        row_rank=ref.product.row_rank.astype(np.int32), col_rank=ref.product.col_rank.astype(np.int32),
        row_degenerate=ref.product.row_degenerate.astype(np.uint8),
        col_degenerate=ref.product.col_degenerate.astype(np.uint8),
        flops=np.int64(rep.flops), case_flops=np.asarray(rep.case_flops, dtype=np.int64),
        max_row_rank=np.array([v.max_row_rank for v in lv], dtype=np.int64),
        max_col_rank=np.array([v.max_col_rank for v in lv], dtype=np.int64),
        case_products=np.array([list(v.case_products) for v in lv], dtype=np.int64),
        max_case_terms=np.array([[v.max_case1_terms, v.max_case2_terms, v.max_case3_terms] for v in lv],
                                dtype=np.int64),
        S=Wv.conj().T @ Y, SA=SA, SB=SB, rows=rows, Yrows=Y[rows], ynorm=np.linalg.norm(Y, axis=0),
    )
    path = os.path.join(ROOT, "tests", "golden", f"full_{name}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **out)
    info = {"name": name, "N": n, "eps": eps, "margin": margin, "flops": int(rep.flops), "oracle_seconds": t_oracle,
            "probe_seconds": t_probe, "threads": threads, "build_seconds": W["build_seconds"],
            "max_rank": int(rep.max_rank()), "bytes": os.path.getsize(path)}
    print(json.dumps(info), flush=True)
    return info


def main():
    from bench import host_cores
    names = sys.argv[1:] or ["cfg2", "cfg3", "cfg5s"]
    infos = [make(n, host_cores()) for n in names]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fixtures.json"), "w") as f:
        json.dump(infos, f, indent=1)


if __name__ == "__main__":
    main()
