"""One device-resident factorization of a named workload (profiling/debug aid):
python tools/one_factor.py [C4] [reps] [lowmem].  RPC_DEBUG_TIMING=1 prints per-launch update TF/s."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl, _lib as L
w = wl.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lowmem = len(sys.argv) > 3 and sys.argv[3] == "lowmem"
x = torch.from_numpy(np.ascontiguousarray(w.points())).cuda()
ctx = api.Context(0)
cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
spec = api.KernelSpec(w.kernel, w.sigma)
for i in range(reps):
    fn = api.accelerated_rpcholesky_lowmem_device if lowmem else api.accelerated_rpcholesky_device
    r = fn(x.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR, spec, cfg, ctx)
    t = r.timing
    print(f"{w.name} rep {i}: factorize {t['factorize_ms']:.2f} ms update {t['update_ms']:.2f} ms "
          f"({t['update_flops'] / t['update_ms'] / 1e9:.2f} TF/s) rank {r.rank}", flush=True)
    r.free()
ctx.close()
