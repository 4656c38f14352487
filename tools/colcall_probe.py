"""Debug aid: device time of rpc_kernel_columns (single launch) vs bench_column_throughput."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl
w = wl.CONFIGS["C4"]
ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
ctx = api.Context(0)
rng = np.random.default_rng(0)
for m in (27, 70, 91, 102, 116):
    cols = rng.integers(0, w.n, m)
    ko.columns(cols, ctx, return_ms=True)
    ts = [ko.columns(cols, ctx, return_ms=True)[1] for _ in range(3)]
    print(f"m={m}: columns() {min(ts) * 1e3:.0f} us  {8 * w.n * m / (min(ts) * 1e-3) / 1e9:.0f} GB/s")
ctx.close()
