"""One C4 factorization from device-resident points (a short command for ncu captures:
ncu -k regex:update_kernel -s 9 -c 1 ... python tools/one_c4.py  -> the round-9 update)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_03969_b200 import _lib as L  # noqa: E402
from paper_2410_03969_b200 import api, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = workloads.CONFIGS[name]
ctx = api.Context(0)
xd = torch.from_numpy(np.ascontiguousarray(w.points())).cuda()
r = api.accelerated_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR,
                                      api.KernelSpec(w.kernel, w.sigma),
                                      api.RunConfig.until_rank(w.k, w.b, w.seed), ctx)
print(name, "rank", r.rank, "factorize_ms", r.timing["factorize_ms"])
r.free()
