"""KRR kernel_matvec probe (debug aid)."""
import math, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl
n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000, 10
x = wl.gen_c1(n, d, 0)
ko = api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(d)))
v = np.random.default_rng(0).standard_normal(n)
for i in range(3):
    t0 = time.perf_counter()
    api.kernel_matvec(ko, v)
    print(f"matvec n={n}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
