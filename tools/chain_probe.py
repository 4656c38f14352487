"""Per-stage device timeline of the round loop (RPC_DEBUG_CHAIN=1: an event after every
stage; the time between consecutive events is charged to the later stage, launch gaps
included).  Usage: RPC_DEBUG_CHAIN=1 python tools/chain_probe.py C4 [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_03969_b200 import _lib as L  # noqa: E402
from paper_2410_03969_b200 import api, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = workloads.CONFIGS[name]
ctx = api.Context(0)
xd = torch.from_numpy(np.ascontiguousarray(w.points())).cuda()
for i in range(reps):
    print(f"--- {name} run {i}", file=sys.stderr, flush=True)
    r = api.accelerated_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR,
                                          api.KernelSpec(w.kernel, w.sigma),
                                          api.RunConfig.until_rank(w.k, w.b, w.seed), ctx)
    print(name, "rank", r.rank, "factorize_ms", round(r.timing["factorize_ms"], 3),
          "update_ms", round(r.timing["update_ms"], 3), file=sys.stderr, flush=True)
    r.free()
