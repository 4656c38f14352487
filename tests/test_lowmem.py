"""Low-memory variant: accelerated_rpcholesky_lowmem (rpcholesky.hpp:408-485).

Pins: the C restatement (oracle/rpc_oracle.c rpo_accelerated_rpcholesky_lowmem) must
reproduce the reference's own lowmem run bit for bit (fixtures tests/golden/ref_lowmem_*.npz
made by tests/golden/make_ref_fixtures.py from oracle/_ref, and pyref directly where it is
built).  The CUDA path (rpc_accelerated_rpcholesky_lowmem through the C-ABI) must give the
identical pivots and trace, and chol_factor / residual_diag at the bars below.  The GPU
forms the proposals' factor rows as A(S', S) L^{-T} with an explicit L^{-1} and the
diagonal update as one product A(R, S_all) W^T (lowmem_impl.cuh), where the reference
triangular-solves per row chunk; both are the same quantity, rounded differently.

Bars: pivots / proposals / accepted counts identical; chol_factor relative Frobenius
error <= 1e-10; residual diagonal max abs error <= 1e-8 (the reference's own bar for
lowmem vs standard, test_rpcholesky.cpp:265-280); captured_sq relative <= 1e-10.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as po
import pyref
from paper_2410_03969_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["c1", "c3s", "c5s"]
CHOL_TOL = 1e-10
U_TOL = 1e-8


def load(name):
    z = np.load(os.path.join(GOLDEN, f"ref_lowmem_{name}.npz"))
    gen, n, d, kern, sigma, k, b, seed = [str(v) for v in z["config"]]
    x = wl.GENERATORS[gen](int(n), int(d), 0)
    return z, x, kern, float(eval(sigma)), int(k), int(b), int(seed)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def compare(z, pivots, proposed, acc_counts, exhausted, surplus, chol, resid, exact=False):
    assert np.array_equal(pivots, z["pivots"])
    assert np.array_equal(np.array(proposed), z["proposed"])
    assert np.array_equal(np.array(acc_counts), z["accepted_counts"])
    assert bool(exhausted) == bool(z["rank_exhausted"]) and int(surplus) == int(z["surplus"])
    if exact:
        assert np.array_equal(chol, z["chol"])
        assert np.array_equal(resid, z["residual_diag"])
    else:
        assert rel(chol, z["chol"]) <= CHOL_TOL
        assert np.max(np.abs(resid - z["residual_diag"])) <= U_TOL


# ------------------------------------------------------------------ CPU pins
@pytest.mark.parametrize("name", CASES)
def test_oracle_lowmem_reproduces_reference_fixture(name):
    z, x, kern, sigma, k, b, seed = load(name)
    o = po.Oracle(x=x, kernel=kern, sigma=sigma, n_threads=8)
    r = po.accelerated_rpcholesky_lowmem(o, block_size=b, target_rank=k, seed=seed)
    assert r.factor is None
    compare(z, r.pivots, r.proposed, [len(a) for a in r.accepted], r.rank_exhausted, r.surplus,
            r.chol, r.residual_diag, exact=True)


@pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kern,dist,mode", [("gaussian", "gram", "until_rank"),
                                            ("gaussian", "direct", "fixed_rounds"),
                                            ("l1laplace", "direct", "until_rank")])
def test_oracle_lowmem_identical_to_reference(kern, dist, mode):
    x = wl.gen_c2(2500, 6, 3)
    kw = dict(block_size=17, seed=5, mode=mode)
    kw.update(rounds=5) if mode == "fixed_rounds" else kw.update(target_rank=80)
    a = pyref.accelerated_rpcholesky_lowmem_kernel(x, kern, 2.0, dist=dist, **kw)
    r = po.accelerated_rpcholesky_lowmem(po.Oracle(x=x, kernel=kern, sigma=2.0, dist=dist), **kw)
    assert np.array_equal(a.pivots, r.pivots)
    assert np.array_equal(a.chol, r.chol)
    assert np.array_equal(a.residual_diag, r.residual_diag)
    assert [len(v) for v in a.accepted] == [len(v) for v in r.accepted]
    assert a.surplus == r.surplus and a.rank_exhausted == r.rank_exhausted


def test_oracle_lowmem_equals_standard_pivots():  # test_rpcholesky.cpp:265-280
    x = wl.gen_c1(3000, 5, 2)
    o = po.Oracle(x=x, kernel="gaussian", sigma=1.5)
    s = po.accelerated_rpcholesky(o, block_size=25, target_rank=150, seed=1)
    lm = po.accelerated_rpcholesky_lowmem(o, block_size=25, target_rank=150, seed=1)
    assert np.array_equal(s.pivots, lm.pivots)
    assert np.max(np.abs(s.residual_diag - lm.residual_diag)) <= 1e-8


def test_oracle_lowmem_errors():
    o = po.Oracle(x=wl.gen_c1(50, 2, 0), kernel="gaussian", sigma=1.0)
    with pytest.raises(ValueError, match="block size"):
        po.accelerated_rpcholesky_lowmem(o, block_size=0, target_rank=3)


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def ctx():
    from paper_2410_03969_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def run_both(ctx, x, kernel, sigma, k=None, b=8, seed=0, rounds=None, replay=False, dist=None,
             stop_tol=0.0):
    from paper_2410_03969_b200 import api
    if rounds is not None:
        cfg = api.RunConfig.fixed_rounds(rounds, b, seed)
        okw = dict(mode="fixed_rounds", rounds=rounds)
    else:
        cfg = api.RunConfig.until_rank(k, b, seed)
        okw = dict(target_rank=k)
    cfg.replay_scan = replay
    cfg.stop_tol = stop_tol
    g = api.accelerated_rpcholesky_lowmem(api.KernelOracle(x, api.KernelSpec(kernel, sigma), dist),
                                          cfg, ctx)
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma, dist=dist, n_threads=8)
    r = po.accelerated_rpcholesky_lowmem(o, block_size=b, seed=seed, stop_tol=stop_tol, **okw)
    return g, r


def assert_parity(g, r):
    assert np.array_equal(g.pivots, r.pivots)
    assert len(g.proposed) == len(r.proposed)
    for a, bb in zip(g.proposed, r.proposed):
        assert np.array_equal(a, bb)
    for a, bb in zip(g.accepted, r.accepted):
        assert np.array_equal(a, bb)
    assert g.rank_exhausted == r.rank_exhausted
    assert g.surplus == r.surplus
    if g.rank:
        assert rel(g.chol_factor, r.chol) <= CHOL_TOL
    assert np.max(np.abs(g.residual_diag - r.residual_diag)) <= U_TOL
    assert abs(g.captured_sq - r.captured_sq) <= 1e-10 * max(1.0, r.captured_sq)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("replay", [False, True])
def test_gpu_lowmem_matches_reference_fixture(ctx, name, replay):
    from paper_2410_03969_b200 import api
    z, x, kern, sigma, k, b, seed = load(name)
    cfg = api.RunConfig.until_rank(k, b, seed)
    cfg.replay_scan = replay
    g = api.accelerated_rpcholesky_lowmem(api.KernelOracle(x, api.KernelSpec(kern, sigma)), cfg, ctx)
    compare(z, g.pivots, g.proposed, [len(a) for a in g.accepted], g.rank_exhausted, g.surplus,
            g.chol_factor, g.residual_diag)


@pytest.mark.gpu
def test_gpu_lowmem_gaussian_direct(ctx):
    x = wl.gen_c2(5000, 20, 0)
    g, r = run_both(ctx, x, "gaussian", math.sqrt(20.0), k=150, b=50, dist="direct")
    assert_parity(g, r)


@pytest.mark.gpu
@pytest.mark.parametrize("b", [1, 3, 8, 17])
def test_gpu_lowmem_fixed_rounds_small_blocks(ctx, b):
    x = wl.gen_c1(2000, 4, 7)
    g, r = run_both(ctx, x, "gaussian", 1.0, rounds=6, b=b, seed=11)
    assert_parity(g, r)


@pytest.mark.gpu
def test_gpu_lowmem_exact_rank_and_exhaustion(ctx):
    base = wl.gen_c1(5, 3, 1) * 2.0
    x = np.repeat(base, 40, axis=0)
    g, r = run_both(ctx, x, "gaussian", 1.0, k=5, b=2)
    assert np.array_equal(g.pivots, r.pivots)
    g, r = run_both(ctx, np.zeros((50, 3)), "gaussian", 1.0, k=10, b=3)
    assert g.rank_exhausted and r.rank_exhausted and g.rank == r.rank == 1
    assert_parity(g, r)


@pytest.mark.gpu
def test_gpu_lowmem_stop_tol_and_tiny(ctx):
    x = wl.gen_c1(3000, 2, 5)
    g, r = run_both(ctx, x, "gaussian", 1.0, k=500, b=10, stop_tol=0.05)
    assert g.rank < 500
    assert_parity(g, r)
    g, r = run_both(ctx, np.array([[0.0], [1.0], [3.0]]), "gaussian", 1.0, k=3, b=2)
    assert_parity(g, r)


@pytest.mark.gpu
def test_gpu_lowmem_equals_standard_gpu(ctx):
    from paper_2410_03969_b200 import api
    x = wl.gen_c1(20000, 10, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(10.0)))
    cfg = api.RunConfig.until_rank(200, 40, 0)
    s = api.accelerated_rpcholesky(ko, cfg, ctx)
    lm = api.accelerated_rpcholesky_lowmem(ko, cfg, ctx)
    assert np.array_equal(s.pivots, lm.pivots)
    assert np.max(np.abs(s.residual_diag - lm.residual_diag)) <= 1e-8
    assert rel(lm.chol_factor, s.chol_factor) <= 1e-10
    with pytest.raises(ValueError, match="not stored"):
        lm.factor


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 3, 7])
def test_gpu_lowmem_virtual_shards_p_invariance(p):
    from paper_2410_03969_b200 import api
    x = wl.gen_c3(12000, 50, 0)
    ko = api.KernelOracle(x, api.KernelSpec("l1laplace", 5.0))
    cfg = api.RunConfig.until_rank(300, 120, 0)
    g1 = api.accelerated_rpcholesky_lowmem(ko, cfg, api.Context(0))
    gp = api.accelerated_rpcholesky_lowmem(ko, cfg, api.Context(0, virtual_shards=p))
    assert np.array_equal(g1.pivots, gp.pivots)
    assert np.array_equal(g1.chol_factor, gp.chol_factor)      # bitwise
    assert np.array_equal(g1.residual_diag, gp.residual_diag)  # bitwise
    assert g1.captured_sq == gp.captured_sq


@pytest.mark.gpu
def test_gpu_lowmem_invalid_arguments(ctx):
    from paper_2410_03969_b200 import api
    x = wl.gen_c1(100, 3, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", 1.0))
    with pytest.raises(ValueError, match="block size"):
        api.accelerated_rpcholesky_lowmem(ko, api.RunConfig(block_size=0, target_rank=3), ctx)
    wide = api.KernelOracle(wl.gen_c1(100, 200, 0), api.KernelSpec("gaussian", 1.0))
    with pytest.raises(ValueError, match="d <= 128"):
        api.accelerated_rpcholesky_lowmem(wide, api.RunConfig.until_rank(3, 2, 0), ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("b,d,kernel", [(256, 8, "gaussian"), (120, 120, "l1laplace"),
                                        (200, 128, "gaussian")])
def test_gpu_lowmem_extreme_shapes(ctx, b, d, kernel):
    """largest block (two warp columns), largest supported dimension (resident X tile of
    128 coordinates, fewer pipeline stages)."""
    x = wl.gen_c2(5000, d, 6)
    g, r = run_both(ctx, x, kernel, math.sqrt(d), k=400, b=b)
    assert_parity(g, r)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,dist", [("matern32", None), ("matern52", "direct")])
def test_gpu_lowmem_matern(ctx, kernel, dist):
    x = wl.gen_c2(5000, 10, 2)
    g, r = run_both(ctx, x, kernel, 3.0, k=200, b=50, dist=dist)
    assert_parity(g, r)
