"""Calibration of the reference arm's extrapolation (bench.py --impl reference).

Times the reference's own CPU accelerated_rpcholesky (oracle/_ref: its headers compiled
against the Eigen-API shim, single thread) on the FULL C4 workload once, and on the
bench's bounded sample (first N' rows, same k, b, seed) a few times, on this host.
Writes profiles/r02_reference_calibration_<config>.json, which bench.py quotes next to
its extrapolated value.  Run on the GPU box's host: python tools/reference_calibration.py
"""
from __future__ import annotations

import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    import pyref
    from paper_2410_03969_b200 import workloads
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    n_sample = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    w = workloads.CONFIGS[name]
    assert pyref.available(), "oracle/_ref/libref_rpchol.so missing"
    x = w.points()
    t0 = time.perf_counter()
    r = pyref.accelerated_rpcholesky_kernel(x, w.kernel, w.sigma, block_size=w.b,
                                            target_rank=w.k, seed=w.seed)
    full_s = time.perf_counter() - t0
    rank_full, rounds_full = len(r.pivots), len(r.proposed)
    del r
    xs = x[:n_sample]
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        rs = pyref.accelerated_rpcholesky_kernel(xs, w.kernel, w.sigma, block_size=w.b,
                                                 target_rank=w.k, seed=w.seed)
        ts.append(time.perf_counter() - t0)
    sample_s = statistics.median(ts)
    out = {"config": name, "n": w.n, "k": w.k, "b": w.b, "threads": 1,
           "cpu_model": cpu_model(), "nproc": os.cpu_count(),
           "full_n_s": full_s, "full_rank": rank_full, "full_rounds": rounds_full,
           "n_sample": n_sample, "sample_s": ts, "sample_median_s": sample_s,
           "sample_rank": len(rs.pivots), "sample_rounds": len(rs.proposed),
           "extrapolated_s": sample_s * w.n / n_sample,
           "extrapolation_over_measured": sample_s * w.n / n_sample / full_s}
    path = os.path.join(ROOT, "profiles", f"r02_reference_calibration_{name}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
