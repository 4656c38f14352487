"""Generates tests/golden/ref_*.npz from the REFERENCE's own code (oracle/_ref:
/root/reference/proj/include/rpchol compiled against the Eigen-API shim).

The GPU box has no /root/reference, so these fixtures carry the reference's
answers there: pivots, PivotTrace rounds, rank_exhausted/surplus, chol_factor,
per-column sums and squared norms of the factor, the residual diagonal, and
relative_trace_error, for BASELINE config C1 (full size) and scaled-down
C2/C3-shaped inputs.  `lowmem` fixtures (ref_lowmem_*.npz) carry the reference's
accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485) answers: pivots, trace,
chol_factor and residual diagonal.
`krr` fixtures (ref_krr_*.npz) carry fit_krr + predict (krr.hpp:177-250): coefficients,
PCG report, preconditioner pivots and predictions on a held-out query set.
`baselines` fixtures (ref_block_*.npz, ref_simple_*.npz) carry block_rpcholesky and
simple_rpcholesky (rpcholesky.hpp:206-333).
Run:  python tests/golden/make_ref_fixtures.py [standard|lowmem|krr|baselines|all]
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
    # Matern kernels (kernels.hpp:66-75) through the same KernelOracle path
    "m32s": ("C2", 6000, 8, "matern32", 2.0, 250, 60, 0),
    "m52s": ("C4", 8000, 30, "matern52", 3.0, 300, 120, 0),
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


# fit_krr (krr.hpp:177-224) + predict: (generator, n, d, kernel, sigma, mu, rank, b, seed, tol,
# materialize_threshold).  "lazy" exercises the reference's on-the-fly matvec path (n > 0).
KRR_CASES = {
    "gauss": ("C1", 3000, 10, "gaussian", math.sqrt(10.0), 1e-3, 200, 40, 0, 1e-8, 8192),
    "l1": ("C3", 2500, 8, "l1laplace", 2.0, 1e-2, 150, 30, 1, 1e-8, 8192),
    "lazy": ("C2", 2000, 6, "gaussian", 1.5, 1e-2, 100, 25, 2, 1e-8, 0),
}


def krr_targets(x):
    return np.sin(x[:, 0]) + 0.3 * x[:, 1] - 0.1 * x[:, -1] ** 2


def make_krr():
    for name, (gen, n, d, kern, sigma, mu, rank, b, seed, tol, thr) in KRR_CASES.items():
        x = wl.GENERATORS[gen](n, d, 0)
        q = wl.GENERATORS[gen](257, d, 9)
        r = pyref.fit_krr(x, krr_targets(x), kern, sigma, mu, rank, b, seed, tol, 500, thr, query=q)
        np.savez_compressed(
            os.path.join(HERE, f"ref_krr_{name}.npz"),
            config=np.array([gen, str(n), str(d), kern, repr(sigma), repr(mu), str(rank), str(b),
                             str(seed), repr(tol), str(thr)]),
            coefficients=r["coefficients"], target_mean=np.array(r["target_mean"]),
            iterations=np.array(r["iterations"]), converged=np.array(r["converged"]),
            relative_residuals=r["relative_residuals"],
            relative_residuals_unreg=r["relative_residuals_unreg"], pivots=r["pivots"],
            predictions=r["predictions"])
        print("krr", name, "iters", r["iterations"], "converged", r["converged"])


# block_rpcholesky / simple_rpcholesky (rpcholesky.hpp:206-333): (algo, generator, n, d,
# kernel, sigma, k, b, seed)
BASELINE_CASES = {
    "block_c1": ("block", "C1", 20000, 10, "gaussian", math.sqrt(10.0), 200, 40, 0),
    "block_c3s": ("block", "C3", 6000, 50, "l1laplace", 5.0, 300, 120, 0),
    "simple_c1s": ("simple", "C1", 6000, 10, "gaussian", math.sqrt(10.0), 150, 1, 0),
}


def make_baselines():
    for name, (algo, gen, n, d, kern, sigma, k, b, seed) in BASELINE_CASES.items():
        x = wl.GENERATORS[gen](n, d, 0)
        if algo == "block":
            r = pyref.block_rpcholesky_kernel(x, kern, sigma, block_size=b, target_rank=k, seed=seed)
        else:
            r = pyref.simple_rpcholesky_kernel(x, kern, sigma, k, seed)
        acc_counts = np.array([len(a) for a in r.accepted], np.int64)
        np.savez_compressed(
            os.path.join(HERE, f"ref_{name}.npz"),
            config=np.array([algo, gen, str(n), str(d), kern, repr(sigma), str(k), str(b), str(seed)]),
            pivots=r.pivots, proposed=np.array(r.proposed), accepted_counts=acc_counts,
            rank_exhausted=np.array(r.rank_exhausted), surplus=np.array(r.surplus),
            chol=r.chol, col_sums=r.factor.sum(axis=0), col_sqnorms=(r.factor ** 2).sum(axis=0),
            residual_diag=r.residual_diag, factor_rows_probe=r.factor[:: max(1, n // 64)])
        print(name, "rank", r.factor.shape[1], "rounds", len(r.proposed))


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
    if what in ("krr", "all"):
        make_krr()
    if what in ("baselines", "all"):
        make_baselines()
