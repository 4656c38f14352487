"""Seeded randomized parity sweep over shapes and options (through the C-ABI on a B200).

Each case draws N (not aligned to the 64-row tiles or 4096-row scan chunks), d, the kernel
and distance mode, b, the stopping rule and the seed, and checks the GPU against the C
restatement (oracle/rpc_oracle.c, pinned to the reference in test_reference_pin.py and the
golden fixtures): accelerated (fast and replay scan), low-memory and block variants.
Bars as in test_gpu_parity.py / test_lowmem.py / test_baselines.py.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2410_03969_b200 import workloads as wl

pytestmark = pytest.mark.gpu

KERNELS = [("gaussian", None), ("gaussian", "direct"), ("l1laplace", None), ("matern32", None),
           ("matern52", "direct")]


def draw_case(i):
    rng = np.random.default_rng(1000 + i)
    n = int(rng.integers(40, 9000))
    d = int(rng.choice([1, 2, 3, 7, 16, 17, 31, 64, 100]))
    kernel, dist = KERNELS[int(rng.integers(len(KERNELS)))]
    b = int(rng.choice([1, 2, 5, 16, 33, 64, 120, 200, 256]))
    fixed = bool(rng.integers(2))
    rounds = int(rng.integers(1, 6))
    k = int(rng.integers(1, max(2, min(n, 400))))
    seed = int(rng.integers(0, 2**63))
    gen = ["C1", "C2", "C3", "C5"][int(rng.integers(4))]
    x = wl.GENERATORS[gen](n, d, i)
    sigma = float(math.sqrt(d) * rng.uniform(0.3, 2.0))
    return dict(x=x, kernel=kernel, dist=dist, b=b, fixed=fixed, rounds=rounds, k=k, seed=seed,
                sigma=sigma, n=n)


# Low-dimensional smooth kernels reach their numerical rank within a few hundred pivots.
# Past it, UntilRank would run (in the reference too) until rounding noise is accepted, and
# every new factor column is rounding noise divided by sqrt(noise): the GPU's DMMA Gram sums
# and the oracle's sequential sums then legitimately disagree at 1e-8 (measured on d <= 3).
# stop_tol = 1e-4 (a supported RunConfig field, rpcholesky.hpp:360) keeps every draw in the
# well-posed regime where the 1e-10 factor bar is meaningful; the pivots stay identical
# either way.
STOP_TOL = 1e-4
# RPC_FUZZ_EXTRA=n adds n more draws per variant (a longer sweep than the default suite)
EXTRA = int(os.environ.get("RPC_FUZZ_EXTRA", "0"))


def cfg_of(api, c):
    cfg = (api.RunConfig.fixed_rounds(c["rounds"], c["b"], c["seed"]) if c["fixed"]
           else api.RunConfig.until_rank(c["k"], c["b"], c["seed"]))
    cfg.stop_tol = STOP_TOL
    return cfg


def okw_of(c):
    return (dict(mode="fixed_rounds", rounds=c["rounds"], stop_tol=STOP_TOL) if c["fixed"]
            else dict(target_rank=c["k"], stop_tol=STOP_TOL))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ctx():
    from paper_2410_03969_b200 import api
    c = api.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("i", list(range(24)) + list(range(1000, 1000 + EXTRA)))
def test_fuzz_accelerated(ctx, i):
    from paper_2410_03969_b200 import api
    c = draw_case(i)
    o = po.Oracle(x=c["x"], kernel=c["kernel"], sigma=c["sigma"], dist=c["dist"], n_threads=8)
    r = po.accelerated_rpcholesky(o, block_size=c["b"], seed=c["seed"], **okw_of(c))
    ko = api.KernelOracle(c["x"], api.KernelSpec(c["kernel"], c["sigma"]), c["dist"])
    for replay in (False, True):
        cfg = cfg_of(api, c)
        cfg.replay_scan = replay
        g = api.accelerated_rpcholesky(ko, cfg, ctx)
        assert np.array_equal(g.pivots, r.pivots), (i, replay)
        assert [len(a) for a in g.accepted] == [len(a) for a in r.accepted]
        assert g.rank_exhausted == r.rank_exhausted and g.surplus == r.surplus
        if r.rank:
            assert rel(g.factor, r.factor) <= 1e-10
            assert rel(g.chol_factor, r.chol) <= 1e-10
        assert np.max(np.abs(g.residual_diag - r.residual_diag)) <= 1e-10


@pytest.mark.parametrize("i", list(range(24, 36)) + list(range(2000, 2000 + EXTRA)))
def test_fuzz_lowmem(ctx, i):
    from paper_2410_03969_b200 import api
    c = draw_case(i)
    o = po.Oracle(x=c["x"], kernel=c["kernel"], sigma=c["sigma"], dist=c["dist"], n_threads=8)
    r = po.accelerated_rpcholesky_lowmem(o, block_size=c["b"], seed=c["seed"], **okw_of(c))
    ko = api.KernelOracle(c["x"], api.KernelSpec(c["kernel"], c["sigma"]), c["dist"])
    g = api.accelerated_rpcholesky_lowmem(ko, cfg_of(api, c), ctx)
    assert np.array_equal(g.pivots, r.pivots), i
    assert g.rank_exhausted == r.rank_exhausted and g.surplus == r.surplus
    if r.rank:
        assert rel(g.chol_factor, r.chol) <= 1e-10
    assert np.max(np.abs(g.residual_diag - r.residual_diag)) <= 1e-8


@pytest.mark.parametrize("i", list(range(36, 48)) + list(range(3000, 3000 + EXTRA)))
def test_fuzz_block(ctx, i):
    from paper_2410_03969_b200 import api
    c = draw_case(i)
    o = po.Oracle(x=c["x"], kernel=c["kernel"], sigma=c["sigma"], dist=c["dist"], n_threads=8)
    try:
        r = po.block_rpcholesky(o, block_size=c["b"], seed=c["seed"], **okw_of(c))
    except RuntimeError:
        pytest.skip("reference block Cholesky fails after the diagonal shift for this draw")
    ko = api.KernelOracle(c["x"], api.KernelSpec(c["kernel"], c["sigma"]), c["dist"])
    g = api.block_rpcholesky(ko, cfg_of(api, c), ctx)
    assert np.array_equal(g.pivots, r.pivots), i
    assert g.surplus == r.surplus
    # Block RPCholesky keeps every distinct proposal, so on a low-dimensional kernel one
    # round of b = 200 factors a numerically singular kept block (shifted LLT) and the
    # factor's trailing columns are amplified rounding noise on both sides (measured 1e-7
    # apart on d <= 3) — the ill-conditioning the paper's rejection step removes.  The
    # well-posed factor bar is in test_baselines.py; here: pivots, trace and the error metric.
    if r.rank:
        f2_g, f2_r = float(np.sum(g.factor ** 2)), float(np.sum(r.factor ** 2))
        assert abs(f2_g - f2_r) <= 1e-8 * c["n"]
