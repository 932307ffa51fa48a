#!/usr/bin/env python3
"""Benchmark of the B200 H^2-MMP on the BASELINE.json workload.

A "step" is one accuracy-controlled product C = A*A (h2mmp::mmp,
mmp.cpp:688-691) of the largest single-GPU BASELINE configuration, configs[4]
(default `--config cfg5`): Helmholtz exp(-i kappa r)/(4 pi r), complex128,
N = 2^20 Fibonacci-sphere points of diameter 16 wavelengths, leaf 64,
Chebyshev order growing with the box size in wavelengths, recompressed at 1e-4;
eps = 1e-4.  `--config cfg1..cfg4` run the other BASELINE configurations.

  value : FP64 GFLOP/s = F_alg / device time per product with F_alg = 2 (real)
          or 8 (complex) x MmpReport.flops (the reference's MAC counter,
          mmp.cpp:67-80; identical to the oracle's), operands resident in HBM,
          CUDA events on the library's stream.
  e2e   : same metric through the drop-in C-ABI call h2c_mmp with pinned host
          buffers (H2D of A, D2H of C inside the timed region); the first
          (cold) call of a fresh context is reported next to it.

`--impl reference` times the reference's OWN mmp() (oracle/_ref/libh2ref.so: the
reference's unmodified MMP-path sources compiled against the Eigen-subset shim,
oracle/eigen_shim; single-threaded as the reference is) on the SAME
configuration and N: each step is a consecutive time window of products
running back to back, value = the reference MACs counted in the timed windows /
their wall time.  If that library is missing, the all-cores oracle restatement
(oracle/product_engine.cpp, bit-identical to the reference in ranks and counters)
stands in (kind "port").  Its inputs come from the CPU-only generator
oracle/_build/libh2inputs.so (cached on disk after the first construction:
~12 min for configs[4] on 16 cores); it never maps the B200 library or touches
the GPU.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N, leaf, order, eps, description)
    "cfg1": (4096, 32, 3, 1e-6, "Laplace 1/(4 pi r), N=4096 cloud seed 1, leaf 32, eta 1, Chebyshev order 3 (k=27), eps 1e-6"),
    "cfg2": (65536, 64, 4, 1e-8, "Laplace 1/(4 pi r), N=65536 cloud seed 1, leaf 64, eta 1, Chebyshev order 4 (k=64), eps 1e-8"),
    "cfg4": (262144, 64, 4, 1e-6, "C = A*B on the 64^3 grid (h = 1/65), leaf 64, eta 1: A = 7-point FD Laplacian "
                                  "(6 / -1, exact near field, rank-1 degenerate far field), B = Laplace 1/(4 pi r) "
                                  "Chebyshev order 4 (k=64), eps 1e-6"),
    # configs[3]'s construction on the 48^3 grid: the 64^3 product's live pending couplings alone
    # (two consecutive levels, ~125 GB) exceed one B200's HBM next to A, B and C
    "cfg3": (262144, 32, 3, 1e-6, "16 parallel unit plates (z = 0.1 p) of 128 x 128 panel centroids, Laplace 1/(4 pi r) "
                                  "with self term 2 ln(1+sqrt2)/(pi h), leaf 32, eta 1, Chebyshev order 3 recompressed "
                                  "at 1e-6; C = A*B, B on the centroids with 0.05 h seeded jitter (seed 2) over A's "
                                  "tree/structure; eps 1e-6"),
    "cfg5": (1048576, 64, 0, 1e-4, "Helmholtz exp(-i k r)/(4 pi r), k = 2 pi, complex128, N = 2^20 Fibonacci-sphere "
                                   "points (seeded rotation, seed 3), diameter 16 wavelengths, leaf 64, eta 1, "
                                   "Chebyshev order per level clamp(ceil(1 + 1.2 k h_l), 3, 9) recompressed at "
                                   "1e-4; C = A*A, eps 1e-4"),
    # configs[4]'s construction at a quarter of the points on a sphere of half the radius (same
    # points per wavelength)
    "cfg5s": (262144, 64, 0, 1e-4, "configs[4] construction at N = 2^18 on a sphere of diameter 8 wavelengths "
                                   "(same points per wavelength): Helmholtz k = 2 pi, complex128, leaf 64, orders "
                                   "clamp(ceil(1 + 1.2 k h_l), 3, 9), recompressed at 1e-4; C = A*A, eps 1e-4"),
    "cfg4s": (110592, 64, 4, 1e-6, "configs[3] construction on the 48^3 grid (h = 1/49): C = A*B, A = 7-point FD "
                                   "Laplacian, B = Laplace Chebyshev order 4 (k=64), leaf 64, eta 1, eps 1e-6"),
}
DEFAULT_CONFIG = "cfg5"
# CPU baseline of the B200 arm: one warm-up slice + CPU_SLICES slices of CPU_SLICE_S seconds of
# the all-cores oracle product on the same workload (~20 s of CPU work)
CPU_WARM_S, CPU_SLICE_S, CPU_SLICES = 2.0, 5.0, 4
KAPPA = 2.0 * np.pi  # cfg5: wavelength 1


def plate_points(n: int) -> tuple[np.ndarray, float]:
    """16 parallel unit plates z = 0.1 p, m x m panel centroids each (m^2 = n / 16), h = 1/m."""
    m = round((n / 16) ** 0.5)
    h = 1.0 / m
    i, j = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    pl = np.stack([(i.ravel() + 0.5) * h, (j.ravel() + 0.5) * h, np.zeros(m * m)], 1)
    pts = np.concatenate([pl + np.array([0.0, 0.0, 0.1 * p]) for p in range(16)])
    return np.ascontiguousarray(pts), h


def sphere_points(n: int, seed: int = 3) -> np.ndarray:
    """Fibonacci lattice on a sphere of radius 8 sqrt(n / 2^20) (diameter 16 wavelengths at
    N = 2^20; fixed points per wavelength), rotated by a seeded random orthogonal matrix."""
    radius = 8.0 * (n / 2.0 ** 20) ** 0.5
    i = np.arange(n) + 0.5
    phi = np.arccos(1.0 - 2.0 * i / n)
    th = np.pi * (1.0 + 5.0 ** 0.5) * i
    x = radius * np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], 1)
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))
    return np.ascontiguousarray(x @ q.T)


# Chebyshev order cap of configs[4]: the order grows with the box size as clamp(ceil(1 + 1.2 kappa
# h_l), 3, HELM_ORDER_CAP); at N = 2^20 the recompressed (1e-4) ranks of the operand saturate by
# order 9 (max rank per level 46-49 at cap 5, 70-76 at 7, 75-87 at 9: profiles/r02/order_caps_cfg5.txt),
# so higher orders only add constructor cost
HELM_ORDER_CAP = 9


def helmholtz_orders(tree, kappa: float = KAPPA, lo: int = 3, hi: int = HELM_ORDER_CAP) -> np.ndarray:
    """Chebyshev order per level from the largest box half-width h_l in wavelengths."""
    bb = np.asarray(tree.bbox).reshape(-1, 6)
    out = np.full(tree.depth + 1, lo, dtype=np.int32)
    for l in range(tree.depth + 1):
        hl = 0.5 * (bb[tree.level == l, 3:] - bb[tree.level == l, :3]).max()
        out[l] = min(hi, max(lo, int(np.ceil(1.0 + 1.2 * kappa * hl))))
    return out


def grid_points(m: int) -> tuple[np.ndarray, float]:
    """m^3 interior grid of the unit cube, h = 1/(m+1)."""
    h = 1.0 / (m + 1)
    g = np.stack(np.meshgrid(*[np.arange(1, m + 1) * h] * 3, indexing="ij"), -1).reshape(-1, 3)
    return np.ascontiguousarray(g), h


def _operand_cache(cache_dir, name: str, n: int, tree, st):
    """Disk cache of constructed operands for the reference arm (its CPU-only constructor needs
    ~12 min for configs[4] on 16 cores; the driver runs the arm once per N of the scaling run).
    Keyed by the configuration, N and the constructor sources; untimed either way."""
    import hashlib
    from paper_1908_05218_b200 import h2io
    h = hashlib.sha1(repr((name, n, CONFIGS[name], HELM_ORDER_CAP, KAPPA)).encode())
    for src in ("paper_1908_05218_b200/csrc/construct.cpp", "paper_1908_05218_b200/csrc/structure.cpp", "bench.py"):
        with open(os.path.join(ROOT, src), "rb") as f:
            h.update(f.read())
    key = h.hexdigest()[:16]

    def cached(tag: str, make):
        if not cache_dir:
            return make()
        path = os.path.join(cache_dir, f"{name}_{n}_{key}_{tag}.npz")
        if os.path.exists(path):
            try:
                return h2io.load_h2(path, tree, st)
            except Exception:
                pass
        m = make()
        try:
            os.makedirs(cache_dir, exist_ok=True)
            tmp = path + f".{os.getpid()}.tmp.npz"
            h2io.save_h2(tmp, m)
            os.replace(tmp, path)
        except Exception:
            pass
        return m

    return cached


def build_operands(name: str, n: int, cache_dir: str | None = None):
    """(points, tree, structure, A, B) of configuration `name` at N = n points (B is A for C = A*A)."""
    import paper_1908_05218_b200 as P
    _, leaf, order, _, _ = CONFIGS[name]
    if name in ("cfg4", "cfg4s"):
        m = round(n ** (1.0 / 3.0))
        pts, h = grid_points(m)
        tree = P.build_cluster_tree(pts, leaf)
        st = P.build_block_tree(tree, tree, 1.0)
        return pts, tree, st, P.build_fd_laplacian(tree, st, pts, h), P.build_chebyshev(tree, st, pts, order)
    if name == "cfg3":
        pts, h = plate_points(n)
        tree = P.build_cluster_tree(pts, leaf)
        st = P.build_block_tree(tree, tree, 1.0)
        diag = 2.0 * np.log(1.0 + np.sqrt(2.0)) / (np.pi * h)
        A = P.build_chebyshev(tree, st, pts, order, diagonal=diag, eps_recompress=1e-6)
        jit = pts + 0.05 * h * np.random.default_rng(2).uniform(-1.0, 1.0, pts.shape)
        B = P.build_chebyshev(tree, st, jit, order, diagonal=diag, eps_recompress=1e-6)
        return pts, tree, st, A, B
    if name in ("cfg5", "cfg5s"):
        pts = sphere_points(n)
        tree = P.build_cluster_tree(pts, leaf)
        st = P.build_block_tree(tree, tree, 1.0)
        cached = _operand_cache(cache_dir, name, n, tree, st)
        A = cached("A", lambda: P.build_chebyshev(tree, st, pts, helmholtz_orders(tree), kernel="helmholtz",
                                                  kappa=KAPPA, eps_recompress=1e-4))
        return pts, tree, st, A, A
    pts = P.random_cloud(n, 1)  # make_random_cloud (geometry.cpp:39-52)
    tree = P.build_cluster_tree(pts, leaf)
    st = P.build_block_tree(tree, tree, 1.0)
    A = P.build_chebyshev(tree, st, pts, order)
    return pts, tree, st, A, A


def build_workload(name: str, cache_dir: str | None = None):
    n, leaf, order, eps, desc = CONFIGS[name]
    t0 = time.perf_counter()
    pts, tree, st, A, B = build_operands(name, n, cache_dir)
    return dict(name=name, points=pts, tree=tree, structure=st, A=A, B=B, eps=eps, desc=desc,
                build_seconds=time.perf_counter() - t0, n=n, leaf=leaf, order=order)


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def fp64_peak_tflops() -> tuple[float, str]:
    p = os.path.join(ROOT, "profiles", "FP64_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["fp64_dmma_tflops"]), "measured DMMA m8n8k4 (profiles/FP64_PEAKS.json)"
    except Exception:
        return 40.0, "fallback: nominal B200 FP64"


def measured_traffic(kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
    phase's kernel from the committed `ncu --set full` capture (profiles/TRAFFIC.json, written
    by tools/ncu_traffic.py from the .ncu-rep of tools/gpu_round.sh), or None."""
    p = os.path.join(ROOT, "profiles", "TRAFFIC.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t[kernel]
        return float(e["dram_bytes_per_launch"]), e.get("source")
    except Exception:
        return None, None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sliced_oracle(A, B, eps, warm: list[float], timed: list[float], threads: int) -> dict:
    """Consecutive slices of the all-cores oracle product C = A*B (oracle/pyoracle.SlicedProduct):
    untimed warm-up slices, then timed slices; GFLOP/s = F_alg of the MACs counted in the timed
    slices / their wall time."""
    from oracle import pyoracle as O
    import paper_1908_05218_b200.h2c as H
    fpm = 8.0 if A.scalar == H.H2C_COMPLEX else 2.0
    t0 = time.perf_counter()
    S = O.SlicedProduct(A, B, eps, threads)
    setup = time.perf_counter() - t0
    try:
        for w in warm:
            S.step(w)
        secs, macs, per = 0.0, 0, []
        prods = 0
        for t in timed:
            el, m, prods = S.step(t)
            secs += el
            macs += m
            per.append(el)
    finally:
        S.close()
    return {"gflops": fpm * macs / secs / 1e9, "seconds": secs, "macs": macs, "fpm": fpm, "products_done": prods,
            "slice_seconds": per, "setup_seconds": setup}


def sliced_reference(A, B, eps, warm: list[float], timed: list[float]) -> dict:
    """Consecutive time windows of the REFERENCE's own mmp() (oracle/_ref/libh2ref.so: the
    reference's unmodified sources + the Eigen-subset shim) running back to back on the workload;
    GFLOP/s = F_alg of the reference MACs counted in the timed windows / their wall time."""
    from oracle import pyref as R
    import paper_1908_05218_b200.h2c as H
    fpm = 8.0 if A.scalar == H.H2C_COMPLEX else 2.0
    t0 = time.perf_counter()
    S = R.SlicedReference(A, B, eps)
    setup = time.perf_counter() - t0
    try:
        for w in warm:
            S.step(w)
        secs, macs, per, prods, pflops = 0.0, 0, [], 0, 0
        for t in timed:
            el, m, prods, pflops = S.step(t)
            secs += el
            macs += m
            per.append(el)
    finally:
        S.close()
    return {"gflops": fpm * macs / secs / 1e9, "seconds": secs, "macs": macs, "fpm": fpm, "products_done": prods,
            "product_flops": pflops, "slice_seconds": per, "setup_seconds": setup}


def run_reference(args) -> None:
    """Reference arm (rank 0 only): the reference's own CPU mmp() on the same config and N.

    oracle/_ref/libh2ref.so holds the reference's unmodified MMP-path sources compiled here against
    oracle/eigen_shim (Eigen is absent from the image); the reference's product is single-threaded
    (mmp.hpp:58-66, no OpenMP in its build), so it runs on one core with single-threaded BLAS.  If
    that library is missing, the all-cores oracle restatement (bit-identical in ranks/counters,
    tests/test_ref_golden.py) stands in and the line says kind "port"."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1908_05218_b200 import h2c
    from oracle import pyref
    h2c.use_inputs_library()  # CPU-only input generator: this arm never maps the B200 library
    name = args.config
    # the CPU-only constructor of configs[4] takes ~12 min on 16 cores (~100 TFLOP of dense k = 729
    # interpolation couplings per pass): built once per box, then read back from a disk cache
    W = build_workload(name, os.environ.get("H2B_BENCH_CACHE", "/tmp/h2b_bench_cache"))
    if pyref.available():
        cores, kind = 1, "reference"
        r = sliced_reference(W["A"], W["B"], W["eps"], [1.0] * args.warmup, [args.ref_slice] * args.steps)
        what = ("the reference's own mmp() (proj/core/src/mmp.cpp and its callees, unmodified, compiled in "
                "oracle/_ref with the Eigen-subset shim; single-threaded as the reference is, 1-thread BLAS)")
    else:
        cores, kind = host_cores(), "port"
        r = sliced_oracle(W["A"], W["B"], W["eps"], [1.0] * args.warmup, [args.ref_slice] * args.steps, cores)
        what = (f"all-cores oracle products (C++ restatement of mmp.cpp, {cores} threads, bit-identical to 1 "
                f"thread)")
    value = r["gflops"]
    sample = (f"{args.steps} consecutive ~{args.ref_slice:g} s windows (after {args.warmup} x 1 s warm-up windows) "
              f"of {what} running back to back on the same {name} workload at N={W['n']}; {r['macs']:.3e} "
              f"reference MACs in {r['seconds']:.1f} s, {r['products_done']} complete products so far; inputs "
              f"from the CPU-only generator or its disk cache (build / load {W['build_seconds']:.0f} s, conversion "
              f"{r['setup_seconds']:.0f} s, untimed)")
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * r["seconds"] / max(1, args.steps), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if r["fpm"] == 8.0 else "f64", "data": "synthetic",
            "config": {"workload": name, "desc": W["desc"], "N": W["n"], "eps": W["eps"]},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "H2-MMP FP64 GFLOP/s (F_alg = 2 real / 8 complex x MmpReport.flops per product / wall)"


# ---------------------------------------------------------------------------
def max_over_ranks(x: float, dist, device: str) -> float:
    """Max of a per-rank scalar (times are taken as the slowest rank)."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(flops_per_rank: float, world: int, seconds: float) -> float:
    """Whole-job GFLOP/s: every rank runs one product (replicas, weak scaling)."""
    return world * flops_per_rank / seconds / 1e9


def hbm_peak_gbs() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        return 7700.0, "fallback: nominal B200 HBM3e"


def kernel_roofline(e: dict, fpm_exec: float, peak_tf: float, peak_gbs: float) -> dict:
    """Roofline of one profiled (phase, kernel) entry: FP64 tensor bound when its arithmetic
    intensity (executed flops / algorithmic bytes) is above the ridge, HBM bound below."""
    fl = fpm_exec * e["macs"]
    by = e.get("bytes", 0) or 0
    s = e["ms"] * 1e-3
    ridge = peak_tf * 1e12 / (peak_gbs * 1e9)
    ai = fl / by if by else float("inf")
    if ai >= ridge:
        ach = fl / s / 1e12
        return {"bound": "tensor", "achieved": round(ach, 3), "peak": peak_tf, "unit": "TFLOP/s",
                "frac": round(ach / peak_tf, 4), "intensity": round(ai, 2)}
    ach = by / s / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak_gbs, "unit": "GB/s",
            "frac": round(ach / peak_gbs, 4), "intensity": round(ai, 2)}


def run_b200(args) -> None:
    import torch
    import paper_1908_05218_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world)
    else:
        torch.cuda.set_device(local)

    W = build_workload(args.config)
    A, B, eps = W["A"], W["B"], W["eps"]
    ctx = P.Context(local)

    # cold drop-in call on the fresh context: structure plan, arena, upload, product, download
    Ap, _pin = P.pin_matrix(A)
    Bp, _pinb = (Ap, None) if B is A else P.pin_matrix(B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.mmp(Ap, Bp, eps, ctx)
    torch.cuda.synchronize()
    cold_s = time.perf_counter() - t0
    plan_s = res.report.plan_seconds
    del res
    gc.collect()

    dA = P.ResidentOperand(A, ctx)
    dB = dA if B is A else P.ResidentOperand(B, ctx)

    # one product with report (counters, exec MACs) + warm-up
    _, rep = P.mmp_resident(dA, dB, eps, want_report=True)
    for _ in range(max(0, args.warmup - 1)):
        P.mmp_resident(dA, dB, eps)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            P.mmp_resident(dA, dB, eps)
            launches += ctx.kernel_launches()
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, dist, "cuda")
    # F_alg: 2 flops per real MAC, 8 per complex MAC; the tensor pipe
    # executes 3 real MACs per complex MAC (Gauss form, unless H2B_CPLX4M=1): 6 executed flops
    fpm = 8.0 if A.scalar == P.H2C_COMPLEX else 2.0
    fpm_exec = (8.0 if os.environ.get("H2B_CPLX4M") else 6.0) if A.scalar == P.H2C_COMPLEX else 2.0
    flops = fpm * rep.flops
    value = job_throughput(flops, world, ms * 1e-3)

    # roofline of the dominant kernel (and of the next ones): one profiled (untimed, serialised) product
    ctx.set_profile(True)
    P.mmp_resident(dA, dB, eps)
    prof_all = ctx.profile()
    ctx.set_profile(False)
    prof = [e for e in prof_all if not e["name"].startswith(("wall:", "host:"))]
    walls = [e for e in prof_all if e["name"].startswith("wall:")]
    peak, peak_src = fp64_peak_tflops()
    hbm, hbm_src = hbm_peak_gbs()
    prof_ms = sum(e["ms"] for e in prof) if prof else 0.0
    roofline = None
    kernels = []
    if prof:
        top = sorted(prof, key=lambda e: -e["ms"])
        dom = top[0]
        rl = kernel_roofline(dom, fpm_exec, peak, hbm)
        traffic, traffic_src = measured_traffic(f"{args.config}:{dom['name']}")
        roofline = {**rl, "kernel": dom["name"], "launches": dom["launches"],
                    "traffic": traffic, "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic_src,
                    "flops_per_launch": fpm_exec * dom["macs"] / dom["launches"],
                    "alg_bytes_per_launch": (dom.get("bytes", 0) or 0) / dom["launches"],
                    "flops_per_mac_exec": fpm_exec,
                    "peak_source": peak_src if rl["bound"] == "tensor" else hbm_src,
                    "share_of_step": round(dom["ms"] / prof_ms, 4) if prof_ms else None,
                    "pipeline_exec_tflops": round(fpm_exec * rep.flops_exec / (ms * 1e-3) / 1e12, 3),
                    "pipeline_frac": round(fpm_exec * rep.flops_exec / (ms * 1e-3) / 1e12 / peak, 4)}
        for e in top[:10]:
            kernels.append({"kernel": e["name"], "ms": round(e["ms"], 2), "share": round(e["ms"] / prof_ms, 4),
                            **kernel_roofline(e, fpm_exec, peak, hbm)})

    # end-to-end through the drop-in C-ABI call with pinned host buffers (warm context)
    del dA, dB
    gc.collect()
    e2e_times = []
    h2d = d2h = 0
    n_e2e = max(1, min(args.steps, 3))
    last = None
    dev_s = []
    for i in range(n_e2e):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = P.mmp(Ap, Bp, eps, ctx)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        h2d, d2h = res.report.h2d_bytes, res.report.d2h_bytes
        dev_s.append(res.report.device_seconds)
        if i == n_e2e - 1:
            last = res  # kept for eps_rel; earlier results return their pinned buffers to the pool
        del res
        gc.collect()  # (untimed) the pinned result buffer goes back to the pool before the next call
    e2e_s = max_over_ranks(sum(e2e_times) / len(e2e_times), dist, "cuda")
    # accuracy of the product, size-independent: eps_rel = ||C x - A (B x)|| / ||A (B x)|| with the
    # reference's seeded random_vector (metrics.cpp:37-55), exact H^2 MVPs on the device (untimed)
    eps_rel = P.relative_error(A, B, last.product, 1, ctx)
    del last
    gc.collect()
    e2e_value = job_throughput(flops, world, e2e_s)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ctx.close()
        del ctx, Ap, Bp, _pin, _pinb
        gc.collect()
        cores = host_cores()
        c = sliced_oracle(A, B, eps, [CPU_WARM_S], [CPU_SLICE_S] * CPU_SLICES, cores)
        cpu = {"value": round(c["gflops"], 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
               "sample": f"{CPU_SLICES} consecutive ~{CPU_SLICE_S:g} s slices (after a {CPU_WARM_S:g} s warm-up "
                         f"slice) of the all-cores oracle product (C++ restatement of mmp.cpp, {cores} threads) "
                         f"on the same {args.config} workload at N={W['n']}, from the start of the product: "
                         f"{c['macs']:.3e} reference MACs in {c['seconds']:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128" if A.scalar == P.H2C_COMPLEX else "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": W["desc"], "N": W["n"], "eps": eps,
                       "macs_per_step": int(rep.flops), "macs_exec_per_step": int(rep.flops_exec),
                       "flops_per_mac": fpm, "eps_rel": eps_rel, "build_seconds": round(W["build_seconds"], 1),
                       "max_rank": rep.max_rank(),
                       "max_rank_per_level": [int(max(v.max_row_rank, v.max_col_rank)) for v in rep.levels],
                       "l2": "inputs (%.1f GB) >> 126 MB L2" % ((A.values.nbytes + (0 if B is A else B.values.nbytes)) / 1e9),
                       "parallelism": f"replicas{world}"},
            "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "seconds": round(e2e_s, 4),
                    "device_seconds_inside": round(sum(dev_s) / len(dev_s), 4),
                    "cold_seconds": round(cold_s, 3), "plan_seconds": round(plan_s, 3),
                    "cold_value": round(job_throughput(flops, world, cold_s), 3)},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
        }
        if args.profile:
            line["profile"] = sorted(prof, key=lambda e: -e["ms"])[:25]
            line["profile_sum_ms"] = round(prof_ms, 3)
            line["phase_wall_ms"] = {e["name"][5:]: round(e["ms"], 2) for e in walls}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def spawn_replicas(args) -> int:
    """`--gpus N` without a launcher: run N replicas (one process per GPU) under torchrun."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-slice", type=float, default=6.0, help="seconds per reference-arm step (oracle slice)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_replicas(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
