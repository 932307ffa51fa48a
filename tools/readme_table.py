"""Results table of README.md from committed bench lines.

Usage: python tools/readme_table.py cfg5=profiles/r02/bench_cfg5_s8.json cfg2=... [reference=...]
"""
import json
import sys

NAMES = {
    "cfg5": "configs[4] cfg5 (bench default): Helmholtz sphere, N=2²⁰, complex128, orders ≤ 9, ε=1e-4",
    "cfg2": "configs[1] cfg2: N=65,536 cloud, leaf 64, k=64, ε=1e-8",
    "cfg3": "configs[2] cfg3: 16 plates, N=262,144, leaf 32, recompressed, C=A·B, ε=1e-6",
    "cfg4": "configs[3] cfg4: 64³ grid (N=262,144), FD Laplacian × Laplace k=64, ε=1e-6",
    "cfg1": "configs[0] cfg1: N=4,096 cloud, leaf 32, k=27, ε=1e-6",
    "cfg5s": "cfg5s: the cfg5 construction at N=2¹⁸",
}
print("| workload | time / product | GFLOP/s | e2e GFLOP/s | ε_rel (MVP probe) | max rank | dominant kernel vs its roofline |")
print("|---|---|---|---|---|---|---|")
ref = None
for a in sys.argv[1:]:
    k, _, p = a.partition("=")
    d = json.load(open(p))
    if k == "reference":
        ref = d
        continue
    r = d.get("roofline") or {}
    rl = f"{r.get('kernel', '')}: {r.get('achieved')} {r.get('unit')} = {r.get('frac')} of the {r.get('bound')} peak" if r else ""
    print(f"| {NAMES[k]} | {d['ms_per_step'] / 1e3:.3f} s | {d['value']:,.0f} | {d['e2e']['value']:,.0f} | "
          f"{d['config']['eps_rel']:.1e} | {d['config']['max_rank']} | {rl} |")
    if d.get("cpu_baseline"):
        c = d["cpu_baseline"]
        print(f"| ↳ all-cores oracle beside it ({c['cores']} threads, same config and N) | | {c['value']:,.0f} | | | | |")
if ref:
    print(f"| ↳ `--impl reference`: the reference's own `mmp()`, 1 thread, same config and N | | {ref['value']:,.1f} | | | | |")
