"""Run one product of a Chebyshev workload with per-phase profiling (debug aid)."""
import sys, time
sys.path.insert(0, "/root/repo")
import paper_1908_05218_b200 as P
n = int(sys.argv[1]); leaf = int(sys.argv[2]); order = int(sys.argv[3]); eps = float(sys.argv[4])
pts = P.random_cloud(n, 1)
t = P.build_cluster_tree(pts, leaf); s = P.build_block_tree(t, t, 1.0)
A = P.build_chebyshev(t, s, pts, order)
ctx = P.Context(0)
ctx.set_profile(True)
t0 = time.time()
r = P.mmp(A, A, eps, ctx)
print("ok", n, time.time() - t0, "flops", r.report.flops, "maxrank", r.report.max_rank(), "dev", r.report.device_seconds,
      "ranks", [(l.max_row_rank, l.max_col_rank) for l in r.report.levels], flush=True)
r = P.mmp(A, A, eps, ctx)  # warm second run
prof = [e for e in ctx.profile() if not e["name"].startswith(("wall:", "host:"))]
hosts = [e for e in ctx.profile() if e["name"].startswith("host:")]
print("host phase times (ms):", [(e["name"][5:], round(e["ms"], 1)) for e in hosts])
walls = [e for e in ctx.profile() if e["name"].startswith("wall:")]
print("phase walls (ms):", [(e["name"][5:], round(e["ms"], 1)) for e in walls])
print("second run dev", r.report.device_seconds, "profile sum ms", sum(e["ms"] for e in prof), "entries", len(prof))
agg = {}
for e in prof:
    k = e["name"].split("/")[1]
    agg[k] = agg.get(k, 0) + e["ms"]
print({k: round(v, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])})
for e in sorted(prof, key=lambda e: -e["ms"])[:40]:
    print(e)
