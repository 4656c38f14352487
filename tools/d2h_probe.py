"""Host-link probe for the e2e path (debug aid): pinned D2H GB/s for large blocks, the
device transpose + D2H of rpc_result_factor_copy, and accelerated_rpcholesky_into."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl

dev = torch.device("cuda", 0)
nbytes = 8_960_000_000
src = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
dst = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
for chunk in (64 << 20, 512 << 20, 2 << 30):
    n = chunk // 8
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for o in range(0, src.numel(), n):
        dst[o:o + n].copy_(src[o:o + n], non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H pinned chunk {chunk >> 20} MB: {nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
del src
w = wl.CONFIGS["C4"]
ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
ctx = api.Context(0)
r = api.accelerated_rpcholesky(ko, cfg, ctx)
out = dst[: w.n * r.rank].numpy().reshape((w.n, r.rank), order="F")
r.factor_into(out)
t0 = time.perf_counter()
r.factor_into(out)
dt = time.perf_counter() - t0
print(f"factor_copy (transpose + D2H) {8 * w.n * r.rank / dt / 1e9:.1f} GB/s, {dt * 1e3:.1f} ms")
r.free()
cap = api.factor_capacity(w.n, cfg)
buf = dst[: w.n * cap].numpy().reshape((w.n, cap), order="F")
for i in range(3):
    t0 = time.perf_counter()
    g = api.accelerated_rpcholesky_into(ko, cfg, buf, ctx)
    dt = time.perf_counter() - t0
    print(f"into: {dt * 1e3:.1f} ms  device factorize {g.timing['factorize_ms']:.1f} ms  host total {g.timing['host_total_ms']:.1f}  upload {g.timing['upload_ms']:.1f}")
    g.free()
ctx.close()
