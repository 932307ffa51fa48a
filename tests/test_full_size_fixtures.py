"""Full-size parity of the B200 product against committed CPU-oracle fixtures (default `-m gpu`).

For configs[1] (cfg2, N=65,536, real), configs[2] (cfg3, N=262,144, real, C = A*B) and
configs[4]'s construction at N=2^18 (cfg5s, complex Helmholtz), tests/golden/full_<cfg>.npz holds
the oracle product's ranks, degenerate flags and MmpReport counters and a two-sided random sketch
of C_ref (tools/make_fixtures.py, run once on the GPU box with the all-cores oracle).  Bars
(BASELINE.json north_star): identical block structure, ranks equal unless an eigenvalue lies within
1e-10 of the threshold, identical counters, ||C_gpu - C_ref||_F / ||C_ref||_F <= 10 eps (sketch
estimate and exact rows of C X).  The measured differences go to gpurun_out/fixture_parity.json.
"""
import json
import os

import numpy as np
import pytest

import paper_1908_05218_b200 as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
NAMES = ["cfg2", "cfg3", "cfg5s"]


def _vectors(n, cplx, k):
    X = np.stack([P.random_vector(n, 1000 + s, cplx) for s in range(k)], 1)
    Wv = np.stack([P.random_vector(n, 2000 + s, cplx) for s in range(k)], 1)
    return np.asfortranarray(X), np.asfortranarray(Wv)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    return P.default_context()


@pytest.mark.parametrize("name", NAMES)
def test_full_size_matches_oracle_fixture(ctx, name):
    import bench
    path = os.path.join(GOLDEN, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_fixtures.py {name} on the GPU box")
    fx = np.load(path)
    W = bench.build_workload(name)
    A, B, eps = W["A"], W["B"], W["eps"]
    assert W["n"] == int(fx["N"]) and eps == float(fx["eps"])
    cplx = A.scalar == P.H2C_COMPLEX
    k = fx["S"].shape[0]
    X, Wv = _vectors(W["n"], cplx, k)
    # the operands must be the ones the fixture was made from
    sa = Wv.conj().T @ P.mvp(A, X, ctx)
    assert _rel(sa, fx["SA"]) <= 1e-11, "fixture stale (operand A changed): rerun tools/make_fixtures.py"
    if B is not A:
        sb = Wv.conj().T @ P.mvp(B, X, ctx)
        assert _rel(sb, fx["SB"]) <= 1e-11, "fixture stale (operand B changed): rerun tools/make_fixtures.py"

    got = P.mmp(A, B, eps, ctx)
    C, rep = got.product, got.report
    assert C.tree is A.tree and C.structure is A.structure  # structure preserved (mmp.cpp:25-26)
    ranks_equal = np.array_equal(C.row_rank, fx["row_rank"]) and np.array_equal(C.col_rank, fx["col_rank"])
    Y = P.mvp(C, X, ctx)
    rec = {"N": W["n"], "eps": eps, "margin": float(fx["margin"]), "ranks_equal": bool(ranks_equal),
           "flops_equal": int(rep.flops) == int(fx["flops"]),
           "sketch_rel_diff": _rel(Wv.conj().T @ Y, fx["S"]),
           "rows_rel_diff": _rel(Y[fx["rows"]], fx["Yrows"]),
           "colnorm_rel_diff": _rel(np.linalg.norm(Y, axis=0), fx["ynorm"]),
           "device_seconds": rep.device_seconds, "oracle_seconds": float(fx["oracle_seconds"])}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = os.path.join(ROOT, "gpurun_out", "fixture_parity.json")
    allrec = json.load(open(out)) if os.path.exists(out) else {}
    allrec[name] = rec
    with open(out, "w") as f:
        json.dump(allrec, f, indent=1)

    assert np.array_equal(C.row_degenerate, fx["row_degenerate"])
    assert np.array_equal(C.col_degenerate, fx["col_degenerate"])
    if float(fx["margin"]) > 1e-10:
        assert ranks_equal, rec
        assert rec["flops_equal"], rec
        assert list(rep.case_flops) == list(fx["case_flops"])
        lv = rep.levels
        assert [v.max_row_rank for v in lv] == list(fx["max_row_rank"])
        assert [v.max_col_rank for v in lv] == list(fx["max_col_rank"])
        assert [list(v.case_products) for v in lv] == fx["case_products"].tolist()
        assert [[v.max_case1_terms, v.max_case2_terms, v.max_case3_terms] for v in lv] == fx["max_case_terms"].tolist()
    assert rec["sketch_rel_diff"] <= 10 * eps, rec
    assert rec["rows_rel_diff"] <= 10 * eps, rec
