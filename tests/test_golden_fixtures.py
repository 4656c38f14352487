"""Golden fixtures produced by the reference's own code (tests/golden/ref_*.npz,
see make_ref_fixtures.py): the CPU oracle must reproduce them (CPU test), and
the CUDA path must match them at the north_star bars (GPU test).  These are the
pins that travel to the GPU box, where /root/reference does not exist."""
import math
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2410_03969_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["c1", "c2s", "c3s", "m32s", "m52s"]


def load(name):
    z = np.load(os.path.join(GOLDEN, f"ref_{name}.npz"))
    gen, n, d, kern, sigma, k, b, seed = [str(v) for v in z["config"]]
    x = wl.GENERATORS[gen](int(n), int(d), 0)
    return z, x, kern, float(eval(sigma)), int(k), int(b), int(seed)


def compare(z, pivots, proposed, acc_counts, exhausted, surplus, chol, factor, resid, err):
    assert np.array_equal(pivots, z["pivots"])
    assert np.array_equal(np.array(proposed), z["proposed"])
    assert np.array_equal(np.array(acc_counts), z["accepted_counts"])
    assert bool(exhausted) == bool(z["rank_exhausted"]) and int(surplus) == int(z["surplus"])
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)  # noqa: E731
    assert rel(chol, z["chol"]) <= 1e-10
    assert rel(factor.sum(axis=0), z["col_sums"]) <= 1e-10
    assert rel((factor ** 2).sum(axis=0), z["col_sqnorms"]) <= 1e-10
    n = factor.shape[0]
    assert rel(factor[:: max(1, n // 64)], z["factor_rows_probe"]) <= 1e-10
    assert np.max(np.abs(resid - z["residual_diag"])) <= 1e-10
    assert abs(err - float(z["relative_trace_error"])) <= 1e-8


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_fixture(name):
    z, x, kern, sigma, k, b, seed = load(name)
    o = po.Oracle(x=x, kernel=kern, sigma=sigma, n_threads=8)
    r = po.accelerated_rpcholesky(o, block_size=b, target_rank=k, seed=seed)
    compare(z, r.pivots, r.proposed, [len(a) for a in r.accepted], r.rank_exhausted, r.surplus,
            r.chol, r.factor, r.residual_diag, po.relative_trace_error(o, r.factor))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("replay", [False, True])
def test_gpu_matches_reference_fixture(name, replay):
    from paper_2410_03969_b200 import api
    z, x, kern, sigma, k, b, seed = load(name)
    cfg = api.RunConfig.until_rank(k, b, seed)
    cfg.replay_scan = replay
    g = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec(kern, sigma)), cfg)
    compare(z, g.pivots, g.proposed, [len(a) for a in g.accepted], g.rank_exhausted, g.surplus,
            g.chol_factor, g.factor, g.residual_diag, g.relative_trace_error)
