"""Timing / sweep count of the device truncation on random PSD Grams (debug aid)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1908_05218_b200 as P
ctx = P.Context(0)
for n in (64, 128, 192, 224, 300):
    rng = np.random.default_rng(n)
    k = (2 * n) // 3
    m = rng.standard_normal((n, k)) * np.logspace(0, -9, k)
    g = m @ m.T
    P.svd_truncate_gram(g, 1e-8, ctx)
    t0 = time.perf_counter()
    for _ in range(3):
        b, d = P.svd_truncate_gram(g, 1e-8, ctx)
    print(n, "rank", b.shape[1], "ms", (time.perf_counter() - t0) / 3 * 1e3, flush=True)
