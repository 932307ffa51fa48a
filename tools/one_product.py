"""One device-resident product of a bench.py workload (short command for ncu captures).

Usage: python tools/one_product.py [cfg]   (cfg1 | cfg2 | cfg4 | cfg4s, default cfg2)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_05218_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
W = bench.build_workload(name)
ctx = P.Context(0)
dA = P.ResidentOperand(W["A"], ctx)
dB = dA if W["B"] is W["A"] else P.ResidentOperand(W["B"], ctx)
_, rep = P.mmp_resident(dA, dB, W["eps"], want_report=True)
print(f"ok {name} flops={rep.flops} flops_exec={rep.flops_exec} max_rank={rep.max_rank()}", flush=True)
