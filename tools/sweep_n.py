"""BASELINE metric "H2-MMP wall time and FP64 GFLOP/s (fraction of the FP64 roofline) vs N" on one
B200: the configs[1] (Laplace cloud, leaf 64, order 4, eps 1e-8) and configs[4] (Helmholtz sphere,
complex, eps 1e-4) constructions over a range of N.  Per point: resident operands, 1 warm-up and
3 timed products (CUDA events on the library stream); F_alg = 2 (real) / 8 (complex) x
MmpReport.flops; executed flops = 2 / 6 (Gauss complex) x flops_exec; fraction of the measured
DMMA peak.  Points that do not fit the HBM are recorded as such.

Usage: python tools/sweep_n.py [out.json] [family:N1,N2,...]"""
import gc
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_05218_b200 as P  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_n.json"
peak, _ = bench.fp64_peak_tflops()
points = [("cfg2", n) for n in (8192, 16384, 32768, 65536, 131072, 262144)] + \
         [("cfg5", n) for n in (16384, 65536, 262144, 1048576)]
if len(sys.argv) > 2:  # e.g. cfg2:65536,131072
    fam, _, ns = sys.argv[2].partition(":")
    points = [(fam, int(x)) for x in ns.split(",")]
rows = []
for name, n in points:
    rec = {"family": name, "N": n, "eps": bench.CONFIGS[name][3]}
    ctx = dA = dB = A = B = None
    gc.collect()  # the previous point's context (and its arena) must be gone
    try:
        t0 = time.perf_counter()
        _, tree, _, A, B = bench.build_operands(name, n)
        rec["build_s"] = round(time.perf_counter() - t0, 1)
        ctx = P.Context(0)
        dA = P.ResidentOperand(A, ctx)
        dB = dA if B is A else P.ResidentOperand(B, ctx)
        _, rep = P.mmp_resident(dA, dB, rec["eps"], want_report=True)
        ts = [P.mmp_resident(dA, dB, rec["eps"])[0] for _ in range(3)]
        t = statistics.median(ts)
        cplx = A.scalar == P.H2C_COMPLEX
        f_alg = (8.0 if cplx else 2.0) * rep.flops
        f_exe = (6.0 if cplx else 2.0) * rep.flops_exec
        rec.update(seconds=round(t, 4), gflops=round(f_alg / t / 1e9, 1), exec_tflops=round(f_exe / t / 1e12, 2),
                   frac_of_dmma_peak=round(f_exe / t / 1e12 / peak, 3), depth=tree.depth, max_rank=rep.max_rank(),
                   macs=int(rep.flops), macs_exec=int(rep.flops_exec))
    except Exception as e:  # e.g. device memory
        rec["error"] = str(e)[:200]
    ctx = dA = dB = A = B = None
    rows.append(rec)
    print(json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)
