"""Kernel-column throughput probe (debug aid): bench_column_throughput on C4's points."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl
w = wl.CONFIGS["C4"]
ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
bs = [int(a) for a in sys.argv[1:]] or [120]
for r in api.bench_column_throughput(ko, bs, 0):
    print(r)
