"""Standalone kernel columns with the Gram on the int8 tensor cores (i8cols.cu; Gaussian /
Matérn Gram mode, d <= 32): against the C restatement of oracle.hpp:71-90 and against the
FP64 DMMA columns kernel (RPC_NO_I8COLS=1) on the same inputs."""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import pyoracle as po  # noqa: E402
from paper_2410_03969_b200 import api  # noqa: E402
from paper_2410_03969_b200 import workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = api.Context(0)
    yield c
    c.close()


def fp64_columns(ko, cols, ctx):
    os.environ["RPC_NO_I8COLS"] = "1"
    try:
        return ko.columns(cols, ctx)
    finally:
        del os.environ["RPC_NO_I8COLS"]


@pytest.mark.parametrize("n,d,kernel", [(1000, 1, "gaussian"), (70001, 30, "gaussian"),
                                        (4099, 32, "gaussian"), (5000, 17, "matern52"),
                                        (333, 8, "matern32")])
def test_i8cols_matches_oracle_and_fp64(ctx, n, d, kernel):
    x = wl.gen_c4(n, d, 3) if d > 1 else wl.gen_c1(n, 1, 3)
    sigma = math.sqrt(d) * 0.8
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma, dist="gram", n_threads=8)
    ko = api.KernelOracle(x, api.KernelSpec(kernel, sigma), "gram")
    rng = np.random.default_rng(n)
    for m in (1, 63, 64, 65, 120, 128, 129, 300):
        cols = rng.integers(0, n, m)
        got = ko.columns(cols, ctx)
        want = o.columns(cols)
        ref = fp64_columns(ko, cols, ctx)
        assert np.max(np.abs(got - want)) <= 1e-13, (m, np.max(np.abs(got - want)))
        assert np.max(np.abs(got - ref)) <= 1e-13, (m, np.max(np.abs(got - ref)))
        assert np.all(got[cols, np.arange(m)] == 1.0)  # same-index pin


def test_i8cols_scaled_rows(ctx):
    """Rows spanning many binades (per-row exponents) and exact zero rows."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((20000, 24)) * np.exp2(rng.integers(-20, 6, (20000, 1)))
    x[::97] = 0.0
    sigma = 4.0
    o = po.Oracle(x=x, kernel="gaussian", sigma=sigma, dist="gram", n_threads=8)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", sigma), "gram")
    cols = np.concatenate([[0, 97, 1], rng.integers(0, 20000, 117)])
    got = ko.columns(cols, ctx)
    assert np.max(np.abs(got - o.columns(cols))) <= 1e-13
    assert np.max(np.abs(got - fp64_columns(ko, cols, ctx))) <= 1e-13


def test_i8cols_bench_rows(ctx):
    """bench_column_throughput Gram rows through the tensor-core kernel (b up to 300)."""
    x = wl.gen_c4(200000, 30, 0)
    rows = api.bench_column_throughput(api.KernelOracle(x, api.KernelSpec("gaussian", 3.0)),
                                       [40, 120, 300], 0, ctx)
    gram = [r for r in rows if r["mode"] == "gram"]
    assert [r["block_size"] for r in gram] == [40, 120, 300]
    for r in gram:
        assert r["output_gbs"] > 0
