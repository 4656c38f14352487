"""Pins the CPU restatement (oracle/rpc_oracle.c) against the reference's OWN
headers compiled here (oracle/_ref, Eigen-API shim), and generates the golden
fixtures the GPU tests compare against on the box (where /root/reference is absent).

Both sides sum in ascending index order, so most quantities agree bitwise; the
tolerances below are the north_star bars, used only where exp()/ordering could
legitimately differ.
"""
import math

import numpy as np
import pytest

import pyoracle as po
import pyref
from paper_2410_03969_b200 import workloads as wl

pytestmark = pytest.mark.skipif(not pyref.available(),
                                reason="oracle/_ref not built (needs /root/reference at build time)")


def random_psd(n, r, seed):
    w = wl.normals(seed, 0, n * r).reshape(r, n).T
    a = w @ w.T
    return 0.5 * (a + a.T)


def test_sample_discrete_identical():
    rng = np.random.default_rng(0)
    for n in (1, 5, 1000, 5000):
        w = rng.random(n)
        w[rng.random(n) < 0.3] = 0.0
        w[-1] = 0.0 if n > 1 else 1.0
        cs = po.cumulative_sums(w)
        want = pyref.sample_discrete(w, 11, 3, 100)
        got = [po.sample_discrete(cs, po.u01(po.splitmix64_draw(11, 3 + j))) for j in range(100)]
        assert list(want) == got


def test_rejection_sweep_identical():
    x = wl.gen_c1(300, 4, 2)
    rng = np.random.default_rng(1)
    for b in (1, 5, 40, 120):
        prop = rng.integers(0, 300, b)
        prop[b // 2:] = prop[: b - b // 2]
        h = pyref.kernel_submatrix(x, "gaussian", 1.1, prop, prop)
        for seed in (0, 9):
            ra, rp, rl = pyref.rejection_sweep(h, prop, seed, 7)
            oa, op, ol = po.rejection_sweep(h, prop, seed, 7)
            assert np.array_equal(ra, oa) and np.array_equal(rp, op)
            assert np.array_equal(rl, ol)


@pytest.mark.parametrize("kernel,dist", [("gaussian", "gram"), ("gaussian", "direct"),
                                         ("l1laplace", None)])
def test_kernel_submatrix_identical(kernel, dist):
    x = wl.gen_c3(400, 7, 3) * 2.0
    o = po.Oracle(x=x, kernel=kernel, sigma=1.3, dist=dist)
    rows = np.arange(400)
    cols = np.array([0, 7, 7, 399, 123])
    a = pyref.kernel_submatrix(x, kernel, 1.3, rows, cols, dist)
    b = o.submatrix(rows, cols)
    assert np.max(np.abs(a - b)) <= 1e-15
    assert np.array_equal(a[cols, np.arange(5)], np.ones(5))


def _same(r, o, ftol=1e-12):
    assert np.array_equal(r.pivots, o.pivots)
    for a, b in zip(r.proposed, o.proposed):
        assert np.array_equal(a, b)
    assert r.rank_exhausted == o.rank_exhausted and r.surplus == o.surplus
    nrm = max(np.linalg.norm(r.factor), 1e-300)
    assert np.linalg.norm(r.factor - o.factor) / nrm <= ftol
    assert np.max(np.abs(r.residual_diag - o.residual_diag)) <= 1e-12


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_accelerated_dense_identical(seed):
    a = random_psd(30, 30, 40 + seed)
    r = pyref.accelerated_rpcholesky_dense(a, block_size=4, target_rank=12, seed=seed)
    o = po.accelerated_rpcholesky(po.Oracle(dense=a), block_size=4, target_rank=12, seed=seed)
    _same(r, o)


def test_accelerated_kernel_c1_scaled():
    x = wl.gen_c1(3000, 10, 0)
    s = math.sqrt(10.0)
    r = pyref.accelerated_rpcholesky_kernel(x, "gaussian", s, block_size=40, target_rank=200)
    o = po.accelerated_rpcholesky(po.Oracle(x=x, kernel="gaussian", sigma=s), block_size=40,
                                  target_rank=200)
    _same(r, o)
    e_r = pyref.relative_trace_error_kernel(x, "gaussian", s, r.factor)
    e_o = po.relative_trace_error(po.Oracle(x=x, kernel="gaussian", sigma=s), o.factor)
    assert abs(e_r - e_o) <= 1e-12


def test_accelerated_kernel_l1_fixed_rounds():
    x = wl.gen_c3(2000, 20, 1)
    r = pyref.accelerated_rpcholesky_kernel(x, "l1laplace", 5.0, block_size=30, mode="fixed_rounds",
                                            rounds=4, seed=5)
    o = po.accelerated_rpcholesky(po.Oracle(x=x, kernel="l1laplace", sigma=5.0), block_size=30,
                                  mode="fixed_rounds", rounds=4, seed=5)
    _same(r, o)


def test_reference_errors_match():
    with pytest.raises(ValueError, match="RunConfig: k, b must be >= 1"):
        pyref.accelerated_rpcholesky_kernel(np.zeros((3, 2)), "gaussian", 1.0, block_size=0,
                                            target_rank=2)
