"""A/B of engine knobs on one resident workload: build the operands once, then for
each configuration (environment overrides) a fresh context, resident upload and
`reps` products; prints the median device seconds per configuration.

  python tools/ab.py N LEAF ORDER EPS 'label:VAR=v,VAR2=w' 'label2:...' ...   (Laplace cloud)
  python tools/ab.py cfg5s 'label:VAR=v' ...                                    (a bench.py config)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_05218_b200 as P

reps = int(os.environ.get("AB_REPS", "3"))
if sys.argv[1].startswith("cfg"):
    import bench
    W = bench.build_workload(sys.argv[1])
    A, B, eps = W["A"], W["B"], W["eps"]
    specs = sys.argv[2:]
else:
    n, leaf, order, eps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
    pts = P.random_cloud(n, 1)
    t = P.build_cluster_tree(pts, leaf)
    s = P.build_block_tree(t, t, 1.0)
    A = B = P.build_chebyshev(t, s, pts, order)
    specs = sys.argv[5:]
KNOBS = ("H2B_AUX_SMS", "H2B_NO_DEFER", "H2B_NO_STRIPS", "H2B_CPLX4M", "H2B_SYM_T64",
         "H2B_NO_STRIPS_SMALL", "H2B_STRIPS_24", "H2B_STRIPS_SMALL_MAX")
for spec in specs:
    label, _, kv = spec.partition(":")
    for k in KNOBS:
        os.environ.pop(k, None)
    for item in filter(None, kv.split(",")):
        k, v = item.split("=")
        os.environ[k] = v
    ctx = P.Context(0)
    dA = P.ResidentOperand(A, ctx)
    dB = dA if B is A else P.ResidentOperand(B, ctx)
    times = []
    for _ in range(reps + 1):
        secs, _ = P.mmp_resident(dA, dB, eps)
        times.append(secs)
    print(f"{label:24s} median {statistics.median(times[1:]):.4f} s  runs {[round(x, 4) for x in times]}", flush=True)
    del dA, dB, ctx
