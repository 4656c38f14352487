"""block_rpcholesky and simple_rpcholesky (rpcholesky.hpp:206-333): the paper's baselines.

Pins: the C restatement (oracle/rpc_oracle.c rpo_block_rpcholesky / rpo_simple_rpcholesky)
reproduces the reference's own runs bit for bit (fixtures tests/golden/ref_block_*.npz,
ref_simple_*.npz from oracle/_ref; pyref directly where built).  The CUDA path
(rpc_block_rpcholesky / rpc_simple_rpcholesky) must give identical pivots and PivotTrace,
and the factor, chol_factor and residual diagonal within the north_star bars (1e-10).
The kept block is factored by the all-accepting sweep (accept iff the residual pivot is
> 0, the LLT success condition), with the reference's one diagonal-shift retry.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as po
import pyref
from paper_2410_03969_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["block_c1", "block_c3s", "simple_c1s"]
TOL = 1e-10


def load(name):
    z = np.load(os.path.join(GOLDEN, f"ref_{name}.npz"))
    algo, gen, n, d, kern, sigma, k, b, seed = [str(v) for v in z["config"]]
    x = wl.GENERATORS[gen](int(n), int(d), 0)
    return z, algo, x, kern, float(eval(sigma)), int(k), int(b), int(seed)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def compare(z, pivots, proposed, acc_counts, exhausted, surplus, chol, factor, resid, exact=False):
    assert np.array_equal(pivots, z["pivots"])
    assert np.array_equal(np.array(proposed), z["proposed"])
    assert np.array_equal(np.array(acc_counts), z["accepted_counts"])
    assert bool(exhausted) == bool(z["rank_exhausted"]) and int(surplus) == int(z["surplus"])
    n = factor.shape[0]
    if exact:
        assert np.array_equal(chol, z["chol"])
        assert np.array_equal(resid, z["residual_diag"])
        assert np.array_equal(factor[:: max(1, n // 64)], z["factor_rows_probe"])
        return
    assert rel(chol, z["chol"]) <= TOL
    assert rel(factor.sum(axis=0), z["col_sums"]) <= TOL
    assert rel((factor ** 2).sum(axis=0), z["col_sqnorms"]) <= TOL
    assert rel(factor[:: max(1, n // 64)], z["factor_rows_probe"]) <= TOL
    assert np.max(np.abs(resid - z["residual_diag"])) <= TOL


def oracle_run(algo, x, kern, sigma, k, b, seed, **kw):
    o = po.Oracle(x=x, kernel=kern, sigma=sigma, n_threads=8, dist=kw.pop("dist", None))
    if algo == "block":
        return po.block_rpcholesky(o, block_size=b, target_rank=k, seed=seed, **kw)
    return po.simple_rpcholesky(o, k, seed)


# ------------------------------------------------------------------ CPU pins
@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_fixture(name):
    z, algo, x, kern, sigma, k, b, seed = load(name)
    r = oracle_run(algo, x, kern, sigma, k, b, seed)
    compare(z, r.pivots, r.proposed, [len(a) for a in r.accepted], r.rank_exhausted, r.surplus,
            r.chol, r.factor, r.residual_diag, exact=True)


@pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")
def test_oracle_identical_to_reference_more_cases():
    x = wl.gen_c2(1500, 5, 3)
    for kw in (dict(mode="fixed_rounds", rounds=4, block_size=64, seed=2),
               dict(block_size=300, target_rank=200, seed=1),       # heavy duplication
               dict(block_size=7, target_rank=50, seed=4, dist="direct")):
        dist = kw.pop("dist", None)
        a = pyref.block_rpcholesky_kernel(x, "gaussian", 2.0, dist=dist, **kw)
        r = po.block_rpcholesky(po.Oracle(x=x, kernel="gaussian", sigma=2.0, dist=dist), **kw)
        assert np.array_equal(a.pivots, r.pivots) and np.array_equal(a.factor, r.factor)
        assert a.surplus == r.surplus
    a = pyref.simple_rpcholesky_kernel(np.zeros((30, 2)), "gaussian", 1.0, 5, 0)
    r = po.simple_rpcholesky(po.Oracle(x=np.zeros((30, 2)), kernel="gaussian", sigma=1.0), 5, 0)
    assert a.rank_exhausted and r.rank_exhausted and a.factor.shape == r.factor.shape


def test_oracle_errors():
    o = po.Oracle(x=wl.gen_c1(20, 2, 0), kernel="gaussian", sigma=1.0)
    with pytest.raises(ValueError, match="need 1 <= k <= N"):
        po.simple_rpcholesky(o, 21, 0)
    with pytest.raises(ValueError, match="block_rpcholesky: block size"):
        po.block_rpcholesky(o, block_size=0, target_rank=3)


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def ctx():
    from paper_2410_03969_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def gpu_run(ctx, algo, x, kern, sigma, k, b, seed, replay=False, dist=None, **kw):
    from paper_2410_03969_b200 import api
    ko = api.KernelOracle(x, api.KernelSpec(kern, sigma), dist)
    if algo == "block":
        if kw.get("mode") == "fixed_rounds":
            cfg = api.RunConfig.fixed_rounds(kw["rounds"], b, seed)
        else:
            cfg = api.RunConfig.until_rank(k, b, seed)
        cfg.replay_scan = replay
        return api.block_rpcholesky(ko, cfg, ctx)
    return api.simple_rpcholesky(ko, k, seed, ctx, replay_scan=replay)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("replay", [False, True])
def test_gpu_matches_reference_fixture(ctx, name, replay):
    z, algo, x, kern, sigma, k, b, seed = load(name)
    g = gpu_run(ctx, algo, x, kern, sigma, k, b, seed, replay)
    compare(z, g.pivots, g.proposed, [len(a) for a in g.accepted], g.rank_exhausted, g.surplus,
            g.chol_factor, g.factor, g.residual_diag)


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(mode="fixed_rounds", rounds=4, b=64, seed=2),
                                dict(b=300 // 2, k=200, seed=1),
                                dict(b=7, k=50, seed=4, dist="direct"),
                                dict(b=400, k=700, seed=5)])  # grouped appends (b > 256)
def test_gpu_block_vs_oracle(ctx, kw):
    x = wl.gen_c2(3000 if kw["b"] > 256 else 1500, 5, 3)
    kw = dict(kw)
    b, seed, dist = kw.pop("b"), kw.pop("seed"), kw.pop("dist", None)
    k = kw.pop("k", 0)
    g = gpu_run(ctx, "block", x, "gaussian", 2.0, k, b, seed, dist=dist, **kw)
    okw = dict(mode="fixed_rounds", rounds=kw["rounds"]) if kw.get("mode") else dict(target_rank=k)
    r = po.block_rpcholesky(po.Oracle(x=x, kernel="gaussian", sigma=2.0, dist=dist),
                            block_size=b, seed=seed, **okw)
    assert np.array_equal(g.pivots, r.pivots)
    assert g.surplus == r.surplus
    assert rel(g.factor, r.factor) <= TOL
    for a, bb in zip(g.accepted, r.accepted):
        assert np.array_equal(a, bb)


@pytest.mark.gpu
@pytest.mark.parametrize("b", [120, 200])
def test_gpu_block_tensor_core_residual(ctx, monkeypatch, b):
    """block_rpcholesky's later rounds on the int8 tensor-core residual (i8gemm.cu; b = 200:
    grouped rounds): same pivots as the FP64 DMMA path and the oracle, factor within TOL."""
    x = wl.gen_c1(30000, 12, 8)
    sigma = math.sqrt(12.0)
    monkeypatch.setenv("RPC_I8_MIN_K", "256")
    monkeypatch.delenv("RPC_NO_I8", raising=False)
    g = gpu_run(ctx, "block", x, "gaussian", sigma, 700, b, 9)
    monkeypatch.setenv("RPC_NO_I8", "1")
    f = gpu_run(ctx, "block", x, "gaussian", sigma, 700, b, 9)
    assert np.array_equal(g.pivots, f.pivots)
    assert rel(g.factor, f.factor) <= TOL
    assert g.timing["tc_int8_ops"] > 0 and f.timing["tc_int8_ops"] == 0
    r = po.block_rpcholesky(po.Oracle(x=x, kernel="gaussian", sigma=sigma, n_threads=8),
                            block_size=b, seed=9, target_rank=700)
    assert np.array_equal(g.pivots, r.pivots)
    assert rel(g.factor, r.factor) <= TOL


@pytest.mark.gpu
def test_gpu_simple_exhaustion_and_errors(ctx):
    from paper_2410_03969_b200 import api
    g = gpu_run(ctx, "simple", np.zeros((30, 2)), "gaussian", 1.0, 5, 1, 0)
    r = po.simple_rpcholesky(po.Oracle(x=np.zeros((30, 2)), kernel="gaussian", sigma=1.0), 5, 0)
    assert g.rank_exhausted and r.rank_exhausted and g.rank == r.rank
    ko = api.KernelOracle(wl.gen_c1(20, 2, 0), api.KernelSpec("gaussian", 1.0))
    with pytest.raises(ValueError, match="need 1 <= k <= N"):
        api.simple_rpcholesky(ko, 21, 0, ctx)
    with pytest.raises(ValueError, match="block_rpcholesky: block size"):
        api.block_rpcholesky(ko, api.RunConfig(block_size=0, target_rank=3), ctx)


@pytest.mark.gpu
def test_gpu_block_duplicate_points(ctx):
    """Distinct indices of identical points make the kept block singular: the reference
    retries with a diagonal shift (rpcholesky.hpp:309-320); the GPU must take the same path."""
    base = wl.gen_c1(40, 3, 5)
    x = np.repeat(base, 25, axis=0)
    try:
        r = po.block_rpcholesky(po.Oracle(x=x, kernel="gaussian", sigma=1.0), block_size=30,
                                target_rank=60, seed=3)
    except RuntimeError as e:
        with pytest.raises(RuntimeError, match="diagonal shift"):
            gpu_run(ctx, "block", x, "gaussian", 1.0, 60, 30, 3)
        assert "diagonal shift" in str(e)
        return
    g = gpu_run(ctx, "block", x, "gaussian", 1.0, 60, 30, 3)
    # after a shifted factorization (pivots ~ sqrt(64 eps)) the residual diagonal carries
    # cond ~ 1e14 amplified rounding, so only the first round is comparable bit for bit
    assert np.array_equal(g.accepted[0], r.accepted[0])
    assert np.array_equal(g.proposed[0], r.proposed[0])
    assert g.rank >= 60


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3])
def test_gpu_block_virtual_shards(p):
    from paper_2410_03969_b200 import api
    x = wl.gen_c1(20000, 10, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(10.0)))
    cfg = api.RunConfig.until_rank(200, 40, 0)
    g1 = api.block_rpcholesky(ko, cfg, api.Context(0))
    gp = api.block_rpcholesky(ko, cfg, api.Context(0, virtual_shards=p))
    assert np.array_equal(g1.pivots, gp.pivots)
    assert np.array_equal(g1.factor, gp.factor)
