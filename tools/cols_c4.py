"""Standalone kernel columns (K5, the COLS update-kernel instantiation) on the C4 points:
blocks of b SplitMix64-drawn columns (rpc_bench_column_throughput, experiment.hpp:344-387).
  python tools/cols_c4.py [b]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_03969_b200 import api, workloads  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 120
w = workloads.CONFIGS["C4"]
ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
for row in api.bench_column_throughput(ko, [b]):
    print(row)
