"""Measurements for the widened rows, one JSON object per line.

  columns     bench_column_throughput (experiment.hpp:344-387) on C4's points: device
              columns/s and kernel-col GB/s per block size and distance mode
  baselines   block_rpcholesky / simple_rpcholesky vs accelerated_rpcholesky on C4's points
              (the paper's speed-up comparison), device factorization time
  krr         fit_krr (krr.hpp:177-224) at N=100k: wall time, PCG iterations, per-iteration
              time and fused-matvec kernel-entry throughput; predict throughput
  rpcf        write_rpcf of the C2 factor (1.8 GB) from the device: wall time and GB/s
  cpu         the reference's own code (oracle/_ref) on bounded samples of the same work,
              single-threaded (the reference's effective parallelism on these paths)

Usage: python tools/bench_components.py [section ...]  (default: all)
"""
import json
import math
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

from paper_2410_03969_b200 import api, workloads as wl  # noqa: E402
from paper_2410_03969_b200 import _lib as L  # noqa: E402


def emit(obj):
    print(json.dumps(obj), flush=True)


def columns(ctx):
    w = wl.CONFIGS["C4"]
    x = w.points()
    ko = api.KernelOracle(x, api.KernelSpec(w.kernel, w.sigma))
    rows = api.bench_column_throughput(ko, [1, 10, 40, 120, 200, 256], 0, ctx)
    for r in rows:
        emit({"section": "columns", "config": f"C4 points N={w.n} d={w.d} gaussian", **r})


def baselines(ctx):
    import torch
    w = wl.CONFIGS["C4"]
    x = w.points()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    spec = api.KernelSpec(w.kernel, w.sigma)
    cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
    runs = {
        "accelerated": lambda: api.accelerated_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d,
                                                                 L.RPC_ROW_MAJOR, spec, cfg, ctx),
        "block": lambda: api.block_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR,
                                                     spec, cfg, ctx),
        "lowmem": lambda: api.accelerated_rpcholesky_lowmem_device(xd.data_ptr(), w.n, w.d, w.d,
                                                                   L.RPC_ROW_MAJOR, spec, cfg, ctx),
        "simple_k300": lambda: api.simple_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d,
                                                            L.RPC_ROW_MAJOR, spec, 300, w.seed, ctx),
    }
    for name, fn in runs.items():
        fn().free()  # warm-up
        ts = []
        for _ in range(3):
            r = fn()
            ts.append(r.timing["factorize_ms"])
            rank, rounds, err = r.rank, len(r.proposed), r.relative_trace_error
            r.free()
        emit({"section": "baselines", "algo": name, "config": f"C4 N={w.n} d={w.d} k={w.k} b={w.b}",
              "device_ms_median": float(np.median(ts)), "rank": rank, "rounds": rounds,
              "relative_trace_error": err})


def krr(ctx):
    n, d = 100_000, 10
    x = wl.gen_c1(n, d, 0)
    t = np.sin(x[:, 0]) + 0.3 * x[:, 1] - 0.1 * x[:, -1] ** 2
    spec = api.KernelSpec("gaussian", math.sqrt(d))
    cfg = api.RunConfig.until_rank(500, 100, 0)
    api.fit_krr(x[:2000], t[:2000], spec, 1e-3, 50, cfg, 1e-6, 20, ctx).model.free()  # warm-up
    t0 = time.perf_counter()
    fit = api.fit_krr(x, t, spec, 1e-3, 500, cfg, 1e-6, 500, ctx)
    wall = time.perf_counter() - t0
    q = wl.gen_c1(20_000, d, 9)
    t1 = time.perf_counter()
    api.predict(fit.model, q)
    pw = time.perf_counter() - t1
    v = np.random.default_rng(0).standard_normal(n)
    ko = api.KernelOracle(x, spec)
    api.kernel_matvec(ko, v, ctx)
    t2 = time.perf_counter()
    api.kernel_matvec(ko, v, ctx)
    mv = time.perf_counter() - t2
    emit({"section": "krr", "config": f"N={n} d={d} gaussian sigma=sqrt(d) mu=1e-3 rank=500 b=100 tol=1e-6",
          "fit_wall_s": wall, "iterations": fit.report.iterations, "converged": fit.report.converged,
          "final_rel_residual": float(fit.report.relative_residuals[-1]) if fit.report.iterations else None,
          "fit_ms_per_iteration": 1e3 * wall / max(1, fit.report.iterations),
          "kernel_matvec_wall_s": mv, "kernel_entries_per_s_matvec": n * n / mv,
          "predict_wall_s_20k": pw, "kernel_entries_per_s_predict": n * 20_000 / pw})
    fit.model.free()


def rpcf(ctx):
    w = wl.CONFIGS["C2"]
    g = api.accelerated_rpcholesky(api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma)),
                                   api.RunConfig.until_rank(w.k, w.b, w.seed), ctx)
    path = os.path.join(tempfile.mkdtemp(), "c2.rpcf")
    g.write_rpcf(path)  # warm-up (staging allocation)
    t0 = time.perf_counter()
    g.write_rpcf(path)
    dt = time.perf_counter() - t0
    size = os.path.getsize(path)
    emit({"section": "rpcf", "config": f"C2 factor N={w.n} k={g.rank}", "bytes": size,
          "wall_s": dt, "gbs": size / dt / 1e9})
    os.remove(path)
    g.free()


def cpu():
    import pyref
    if not pyref.available():
        emit({"section": "cpu", "unavailable": "oracle/_ref not built"})
        return
    w = wl.CONFIGS["C4"]
    ns = 20_000
    x = w.points(ns)
    for name, fn in {
        "accelerated": lambda: pyref.accelerated_rpcholesky_kernel(x, w.kernel, w.sigma, block_size=w.b,
                                                                   target_rank=w.k, seed=w.seed),
        "block": lambda: pyref.block_rpcholesky_kernel(x, w.kernel, w.sigma, block_size=w.b,
                                                       target_rank=w.k, seed=w.seed),
        "lowmem": lambda: pyref.accelerated_rpcholesky_lowmem_kernel(x, w.kernel, w.sigma,
                                                                     block_size=w.b,
                                                                     target_rank=w.k, seed=w.seed),
    }.items():
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        emit({"section": "cpu", "algo": name, "impl": "reference (oracle/_ref, 1 thread)",
              "sample": f"first N'={ns} rows of C4, same k/b/seed", "wall_s": dt,
              "scaled_to_N_s": dt * w.n / ns})
    n = 3000
    xk = wl.gen_c1(n, 10, 0)
    t = np.sin(xk[:, 0]) + 0.3 * xk[:, 1] - 0.1 * xk[:, -1] ** 2
    t0 = time.perf_counter()
    r = pyref.fit_krr(xk, t, "gaussian", math.sqrt(10), 1e-3, 500, 100, 0, 1e-6, 500, 0)
    dt = time.perf_counter() - t0
    emit({"section": "cpu", "algo": "fit_krr (on-the-fly matvec path)", "impl": "reference (oracle/_ref, 1 thread)",
          "sample": f"N={n} d=10, rank 500, tol 1e-6", "wall_s": dt, "iterations": r["iterations"],
          "kernel_entries_per_s_matvec": n * n * r["iterations"] / dt})


def main():
    sections = sys.argv[1:] or ["columns", "baselines", "krr", "rpcf", "cpu"]
    ctx = api.Context(0)
    for s in sections:
        if s == "cpu":
            cpu()
        else:
            globals()[s](ctx)
    ctx.close()


if __name__ == "__main__":
    main()
