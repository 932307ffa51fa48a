"""Per-launch-shape profile of one product of a bench config (H2B_PROF_SHAPES=1): CUDA-event time,
executed MACs and TFLOP/s per (phase, shape), sorted by time.

Usage: python tools/shape_profile.py cfg5s [top]"""
import os
import sys

os.environ["H2B_PROF_SHAPES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1908_05218_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5s"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
W = bench.build_workload(name)
ctx = P.Context(0)
dA = P.ResidentOperand(W["A"], ctx)
dB = dA if W["B"] is W["A"] else P.ResidentOperand(W["B"], ctx)
P.mmp_resident(dA, dB, W["eps"])
ctx.set_profile(True)
P.mmp_resident(dA, dB, W["eps"])
prof = [e for e in ctx.profile() if not e["name"].startswith(("wall:", "host:"))]
fpm = 8.0 if W["A"].scalar == P.H2C_COMPLEX else 2.0
tot = sum(e["ms"] for e in prof)
print(f"# {name}: {len(prof)} entries, {tot:.1f} ms serialised")
for e in sorted(prof, key=lambda e: -e["ms"])[:top]:
    tf = fpm * e["macs"] / (e["ms"] * 1e-3) / 1e12 if e["macs"] else 0.0
    print(f"{e['ms']:8.2f} ms {e['ms'] / tot:6.1%} {tf:6.1f} TF  n={e['launches']:3d}  {e['name']}")
