"""e2e breakdown for accelerated_rpcholesky_into (debug aid)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl
w = wl.CONFIGS["C4"]
xh = torch.from_numpy(np.ascontiguousarray(w.points())).pin_memory().numpy()
ko = api.KernelOracle(xh, api.KernelSpec(w.kernel, w.sigma))
cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
ctx = api.Context(0)
cap = api.factor_capacity(w.n, cfg)
buf = torch.empty(w.n * cap, dtype=torch.float64).pin_memory().numpy().reshape((w.n, cap), order="F")
for i in range(3):
    t0 = time.perf_counter()
    g = api.accelerated_rpcholesky_into(ko, cfg, buf, ctx)
    dt = time.perf_counter() - t0
    print(f"into: {dt * 1e3:.1f} ms  device factorize {g.timing['factorize_ms']:.1f} ms  upload {g.timing['upload_ms']:.1f}  loop {g.timing['host_loop_ms']:.1f}", flush=True)
    g.free()
t0 = time.perf_counter()
g = api.accelerated_rpcholesky(ko, cfg, ctx)
print(f"plain: {(time.perf_counter() - t0) * 1e3:.1f} ms device {g.timing['factorize_ms']:.1f}")
ctx.close()
