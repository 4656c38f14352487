"""bench_column_throughput on the C4 points (debug aid): output GB/s per block size and mode."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03969_b200 import api, workloads as wl
w = wl.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
for r in api.bench_column_throughput(ko, [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1,10,40,120,200,256".split(","))]):
    print(f"b={r['block_size']:4d} {r['mode']:6s} {r['output_gbs']:8.1f} GB/s  {r['wall_ms']:.3f} ms")
