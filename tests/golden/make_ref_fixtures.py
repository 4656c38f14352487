"""Generates tests/golden/ref_*.npz from the REFERENCE's own code (oracle/_ref:
/root/reference/proj/include/rpchol compiled against the Eigen-API shim).

The GPU box has no /root/reference, so these fixtures carry the reference's
answers there: pivots, PivotTrace rounds, rank_exhausted/surplus, chol_factor,
per-column sums and squared norms of the factor, the residual diagonal, and
relative_trace_error, for BASELINE config C1 (full size) and scaled-down
C2/C3-shaped inputs.  `lowmem` fixtures (ref_lowmem_*.npz) carry the reference's
accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485) answers: pivots, trace,
chol_factor and residual diagonal.
Run:  python tests/golden/make_ref_fixtures.py [standard|lowmem|all]
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import pyref  # noqa: E402
from paper_2410_03969_b200 import workloads as wl  # noqa: E402

CASES = {
    # name: (generator, n, d, kernel, sigma, k, b, seed)
    "c1": ("C1", 20000, 10, "gaussian", math.sqrt(10.0), 200, 40, 0),
    "c2s": ("C2", 8000, 20, "gaussian", math.sqrt(20.0), 300, 120, 0),
    "c3s": ("C3", 6000, 50, "l1laplace", 5.0, 300, 120, 0),
}

LOWMEM_CASES = {
    "c1": ("C1", 20000, 10, "gaussian", math.sqrt(10.0), 200, 40, 0),
    "c3s": ("C3", 6000, 50, "l1laplace", 5.0, 300, 120, 0),
    "c5s": ("C5", 6000, 100, "l1laplace", 10.0, 400, 200, 0),
}


def make_lowmem():
    for name, (gen, n, d, kern, sigma, k, b, seed) in LOWMEM_CASES.items():
        x = wl.GENERATORS[gen](n, d, 0)
        r = pyref.accelerated_rpcholesky_lowmem_kernel(x, kern, sigma, block_size=b,
                                                       target_rank=k, seed=seed)
        acc_counts = np.array([len(a) for a in r.accepted], np.int64)
        np.savez_compressed(
            os.path.join(HERE, f"ref_lowmem_{name}.npz"),
            config=np.array([gen, str(n), str(d), kern, repr(sigma), str(k), str(b), str(seed)]),
            pivots=r.pivots, proposed=np.array(r.proposed), accepted_counts=acc_counts,
            rank_exhausted=np.array(r.rank_exhausted), surplus=np.array(r.surplus),
            chol=r.chol, residual_diag=r.residual_diag)
        print("lowmem", name, "rank", len(r.pivots), "rounds", len(r.proposed))


def make_standard():
    for name, (gen, n, d, kern, sigma, k, b, seed) in CASES.items():
        x = wl.GENERATORS[gen](n, d, 0)
        r = pyref.accelerated_rpcholesky_kernel(x, kern, sigma, block_size=b, target_rank=k,
                                                seed=seed)
        err = pyref.relative_trace_error_kernel(x, kern, sigma, r.factor)
        acc_counts = np.array([len(a) for a in r.accepted], np.int64)
        np.savez_compressed(
            os.path.join(HERE, f"ref_{name}.npz"),
            config=np.array([gen, str(n), str(d), kern, repr(sigma), str(k), str(b), str(seed)]),
            pivots=r.pivots, proposed=np.array(r.proposed), accepted_counts=acc_counts,
            rank_exhausted=np.array(r.rank_exhausted), surplus=np.array(r.surplus),
            chol=r.chol, col_sums=r.factor.sum(axis=0), col_sqnorms=(r.factor ** 2).sum(axis=0),
            residual_diag=r.residual_diag, relative_trace_error=np.array(err),
            factor_rows_probe=r.factor[:: max(1, n // 64)])
        print(name, "rank", r.factor.shape[1], "rounds", len(r.proposed), "err", err)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("standard", "all"):
        make_standard()
    if what in ("lowmem", "all"):
        make_lowmem()
