"""Tensor-core residual GEMM (int8 slices) against the FP64 DMMA path on one workload:
pivots, factor difference, trace error, device time.  python tools/i8_check.py [C2|C4|...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_03969_b200 import _lib as L  # noqa: E402
from paper_2410_03969_b200 import api, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = workloads.CONFIGS[name]
ctx = api.Context(0)
xd = torch.from_numpy(np.ascontiguousarray(w.points())).cuda()
spec = api.KernelSpec(w.kernel, w.sigma)
cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
res = {}
for mode in ("dmma", "i8"):
    if mode == "dmma":
        os.environ["RPC_NO_I8"] = "1"
    else:
        os.environ.pop("RPC_NO_I8", None)
    ts = []
    for rep in range(3):
        r = api.accelerated_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR, spec,
                                              cfg, ctx)
        ts.append(r.timing["factorize_ms"])
        if rep < 2:
            r.free()
    res[mode] = (r, ts)
    print(mode, "factorize_ms", [round(t, 2) for t in ts], "rank", r.rank,
          "trace err", r.relative_trace_error, flush=True)
a, b = res["dmma"][0], res["i8"][0]
print("pivots equal:", np.array_equal(a.pivots, b.pivots))
fa, fb = a.factor, b.factor
k = min(fa.shape[1], fb.shape[1])
print("||dF||/||F|| =", np.linalg.norm(fa[:, :k] - fb[:, :k]) / np.linalg.norm(fa[:, :k]),
      " |d trace err| =", abs(a.relative_trace_error - b.relative_trace_error))
