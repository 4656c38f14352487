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
    if w.n * w.k * 8 > 20e9:
        # factor too large to keep two of them: keep its rows at the pivots and the diagonal
        class Keep:
            pass
        kp = Keep()
        kp.pivots, kp.chol_factor, kp.residual_diag = r.pivots.copy(), r.chol_factor.copy(), r.residual_diag.copy()
        kp.relative_trace_error, kp.rank = r.relative_trace_error, r.rank
        r.free()
        r = kp
    res[mode] = (r, ts)
    print(mode, "factorize_ms", [round(t, 2) for t in ts], "rank", r.rank,
          "trace err", r.relative_trace_error, flush=True)
a, b = res["dmma"][0], res["i8"][0]
print("pivots equal:", np.array_equal(a.pivots, b.pivots))
if w.n * w.k * 8 > 20e9:
    # factor too large for the host: its rows at the pivots (chol_factor) and the residual diagonal
    ca, cb = a.chol_factor, b.chol_factor
    print("||d chol||/||chol|| =", np.linalg.norm(ca - cb) / np.linalg.norm(ca),
          " max|du| =", float(np.max(np.abs(a.residual_diag - b.residual_diag))),
          " |d trace err| =", abs(a.relative_trace_error - b.relative_trace_error))
    sys.exit(0)
fa, fb = a.factor, b.factor
k = min(fa.shape[1], fb.shape[1])
print("||dF||/||F|| =", np.linalg.norm(fa[:, :k] - fb[:, :k]) / np.linalg.norm(fa[:, :k]),
      " |d trace err| =", abs(a.relative_trace_error - b.relative_trace_error))
