"""End-to-end (host buffers) timing probe of one bench config through the C-ABI (h2c_mmp):
prints wall time per call; with H2B_E2E_TRACE=1 the library prints its host-side phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_05218_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
W = bench.build_workload(name)
ctx = P.Context(0)
Ap, _pa = P.pin_matrix(W["A"])
Bp, _pb = (Ap, None) if W["B"] is W["A"] else P.pin_matrix(W["B"])
for i in range(4):
    t0 = time.perf_counter()
    r = P.mmp(Ap, Bp, W["eps"], ctx)
    dt = time.perf_counter() - t0
    print(f"{name} call {i}: wall {dt:.3f} s  device {r.report.device_seconds:.3f} s  lib wall {r.report.wall_seconds:.3f} s",
          flush=True)
    del r
