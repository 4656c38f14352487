"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): pivots bit-identical; factor within 1e-10
relative Frobenius error; relative trace error within 1e-8.  Component kernels
are checked at their own natural bars (exact for the sampler and the sweep given
identical inputs; 1e-13 for kernel columns, which differ from the oracle only in
the DMMA summation order of the Gram term and in the last ulp of exp()).
"""
import math

import numpy as np
import pytest

import pyoracle as po
from paper_2410_03969_b200 import api
from paper_2410_03969_b200 import workloads as wl

pytestmark = pytest.mark.gpu

F_TOL = 1e-10       # relative Frobenius error of the factor
TRACE_TOL = 1e-8    # |trace error difference|


@pytest.fixture(scope="module")
def ctx():
    c = api.Context(0)
    yield c
    c.close()


def run_both(x, kernel, sigma, k=None, b=8, seed=0, rounds=None, ctx=None, replay=False,
             dist=None, stop_tol=0.0):
    if rounds is not None:
        cfg = api.RunConfig.fixed_rounds(rounds, b, seed)
        okw = dict(mode="fixed_rounds", rounds=rounds)
    else:
        cfg = api.RunConfig.until_rank(k, b, seed)
        okw = dict(target_rank=k)
    cfg.replay_scan = replay
    cfg.stop_tol = stop_tol
    g = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec(kernel, sigma), dist), cfg,
                                   ctx)
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma, dist=dist, n_threads=8)
    r = po.accelerated_rpcholesky(o, block_size=b, seed=seed, stop_tol=stop_tol, **okw)
    return g, r, o


def assert_parity(g, r, o):
    assert np.array_equal(g.pivots, r.pivots)
    assert len(g.proposed) == len(r.proposed)
    for a, bb in zip(g.proposed, r.proposed):
        assert np.array_equal(a, bb)
    for a, bb in zip(g.accepted, r.accepted):
        assert np.array_equal(a, bb)
    assert g.rank_exhausted == r.rank_exhausted
    assert g.surplus == r.surplus
    f = g.factor
    nrm = np.linalg.norm(r.factor)
    rel = np.linalg.norm(f - r.factor) / nrm if nrm > 0 else np.linalg.norm(f)
    assert rel <= F_TOL, rel
    err_o = po.relative_trace_error(o, r.factor)
    assert abs(g.relative_trace_error - err_o) <= TRACE_TOL
    np.testing.assert_allclose(g.residual_diag, r.residual_diag, rtol=0, atol=1e-10)
    np.testing.assert_allclose(g.chol_factor, r.chol, rtol=0, atol=1e-10)
    return rel


# ---------------------------------------------------------------- components
def test_sample_discrete_replay_bitexact(ctx):
    rng = np.random.default_rng(1)
    for n in (1, 7, 4096, 4097, 10000, 50000):
        u = rng.random(n)
        u[rng.random(n) < 0.3] = 0.0
        if n > 1:
            u[-min(n // 3, 500):] = 0.0  # trailing zero plateau exercises the clamp walk
        if u.sum() == 0:
            u[0] = 1.0
        cs = po.cumulative_sums(u)
        for seed in (0, 3):
            want = [po.sample_discrete(cs, po.u01(po.splitmix64_draw(seed, j))) for j in range(64)]
            got = api.sample_discrete(u, 64, seed, 0, replay=True, ctx=ctx)
            assert list(got) == want


def test_sample_discrete_fast_matches(ctx):
    rng = np.random.default_rng(2)
    for n in (5, 4096, 12289, 100000):
        u = rng.random(n) ** 3
        u[rng.random(n) < 0.2] = 0.0
        cs = po.cumulative_sums(u)
        want = [po.sample_discrete(cs, po.u01(po.splitmix64_draw(9, j))) for j in range(200)]
        got = api.sample_discrete(u, 200, 9, 0, replay=False, ctx=ctx)
        assert list(got) == want
        assert np.all(u[got] > 0.0)   # zero-weight entries are never returned


def test_sample_discrete_clamp_case(ctx):
    # r = 1 - 2^-53 draws may round target up to the total: clamp + plateau walk
    u = np.array([0.0, 3.0, 0.0, 0.0, 0.0])
    for replay in (False, True):
        got = api.sample_discrete(u, 50, 123, 0, replay=replay, ctx=ctx)
        assert np.all(got == 1)


def test_sample_discrete_errors(ctx):
    with pytest.raises(ValueError):
        api.sample_discrete(np.zeros(10), 4, 0, ctx=ctx)


def test_rejection_sweep_bitexact(ctx):
    x = wl.gen_c1(400, 5, 3)
    o = po.Oracle(x=x, kernel="gaussian", sigma=1.3)
    rng = np.random.default_rng(4)
    for b in (1, 2, 17, 40, 120, 200, 256, 300, 700):
        prop = rng.integers(0, 400, b)
        prop[b // 2:] = prop[: b - b // 2]  # duplicates
        h = o.submatrix(prop, prop)
        for seed in (0, 77):
            ga, gp, gl = api.rejection_sample_submatrix(h, prop, seed, 5, ctx=ctx)
            oa, op, ol = po.rejection_sweep(h, prop, seed, 5)
            assert np.array_equal(ga, oa) and np.array_equal(gp, op)
            assert np.array_equal(gl, ol)   # bit-identical given identical H


def test_rejection_sweep_reference_properties(ctx):  # test_rpcholesky.cpp:98-140
    for seed in range(50):
        a, _, l = api.rejection_sample_submatrix(np.array([[0.37]]), [5], seed, 0, ctx=ctx)
        assert list(a) == [5] and l[0, 0] == pytest.approx(math.sqrt(0.37))
        a, _, _ = api.rejection_sample_submatrix(np.full((2, 2), 2.0), [3, 3], seed, 0, ctx=ctx)
        assert len(a) == 1
        a, _, _ = api.rejection_sample_submatrix(np.diag([0.5, 1.5, 0.25]), [0, 1, 2], seed, 0,
                                                 ctx=ctx)
        assert len(a) == 3


@pytest.mark.parametrize("kernel,dist,d", [("gaussian", "gram", 10), ("gaussian", "gram", 37),
                                           ("gaussian", "direct", 12), ("l1laplace", None, 50),
                                           ("l1laplace", None, 3), ("matern32", "gram", 9),
                                           ("matern32", "direct", 20), ("matern52", "gram", 30),
                                           ("matern52", "direct", 5)])
def test_kernel_columns(ctx, kernel, dist, d):
    x = wl.gen_c3(5000, d, 1) * 3.0
    sigma = math.sqrt(d) * 0.7
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma, dist=dist, n_threads=8)
    ko = api.KernelOracle(x, api.KernelSpec(kernel, sigma), dist)
    rng = np.random.default_rng(5)
    for m in (1, 8, 9, 64, 120, 129, 200, 256, 300):
        cols = rng.integers(0, 5000, m)
        got = ko.columns(cols, ctx)
        want = o.columns(cols)
        assert np.max(np.abs(got - want)) <= 1e-13, (m, np.max(np.abs(got - want)))
        # same-index pin: the pivot's own entry is exactly kappa(x, x) = 1
        assert np.all(got[cols, np.arange(m)] == 1.0)


def test_kernel_columns_colmajor_input(ctx):
    x = np.asfortranarray(wl.gen_c1(3000, 6, 2))
    o = po.Oracle(x=x, kernel="gaussian", sigma=2.0)
    got = api.KernelOracle(x, api.KernelSpec("gaussian", 2.0)).columns([0, 5, 2999], ctx)
    assert np.max(np.abs(got - o.columns([0, 5, 2999]))) <= 1e-13


# ----------------------------------------------------------- full algorithm
def test_c1_small_gaussian_parity(ctx):
    x = wl.gen_c1(4000, 10, 0)
    g, r, o = run_both(x, "gaussian", math.sqrt(10.0), k=200, b=40, ctx=ctx)
    assert g.rank >= 200
    assert_parity(g, r, o)


def test_c1_full_parity(ctx):
    w = wl.CONFIGS["C1"]
    x = w.points()
    g, r, o = run_both(x, w.kernel, w.sigma, k=w.k, b=w.b, seed=w.seed, ctx=ctx)
    assert_parity(g, r, o)


def test_c1_replay_mode_parity(ctx):
    w = wl.CONFIGS["C1"]
    x = w.points(8000)
    g, r, o = run_both(x, w.kernel, w.sigma, k=w.k, b=w.b, ctx=ctx, replay=True)
    assert_parity(g, r, o)


def test_l1_parity(ctx):
    x = wl.gen_c3(6000, 50, 0)
    g, r, o = run_both(x, "l1laplace", 5.0, k=300, b=120, ctx=ctx)
    assert_parity(g, r, o)


def test_gaussian_direct_parity(ctx):
    x = wl.gen_c2(5000, 20, 0)
    g, r, o = run_both(x, "gaussian", math.sqrt(20.0), k=150, b=50, ctx=ctx, dist="direct")
    assert_parity(g, r, o)


def test_large_block_parity(ctx):  # b = 200 exercises the 64-row tile variant
    x = wl.gen_c5(6000, 100, 0)
    g, r, o = run_both(x, "l1laplace", 10.0, k=400, b=200, ctx=ctx)
    assert_parity(g, r, o)


@pytest.mark.parametrize("b", [1, 3, 8, 17])
def test_fixed_rounds_and_small_blocks(ctx, b):
    x = wl.gen_c1(2000, 4, 7)
    g, r, o = run_both(x, "gaussian", 1.0, rounds=6, b=b, seed=11, ctx=ctx)
    assert_parity(g, r, o)
    assert all(len(a) >= 1 for a in g.accepted)   # first proposal always accepted


def test_exact_rank_termination(ctx):  # test_rpcholesky.cpp:199-212
    base = wl.gen_c1(5, 3, 1) * 2.0
    x = np.repeat(base, 40, axis=0)          # kernel matrix of exact rank 5
    for kernel in ("gaussian", "l1laplace"):
        g, r, o = run_both(x, kernel, 1.0, k=5, b=2, ctx=ctx)
        assert np.array_equal(g.pivots, r.pivots)
        assert g.relative_trace_error <= 1e-9


def test_rank_exhausted_flag(ctx):  # rpcholesky.hpp:356-359
    x = np.zeros((50, 3))                    # all-ones kernel matrix: rank 1, u -> 0 exactly
    g, r, o = run_both(x, "gaussian", 1.0, k=10, b=3, ctx=ctx)
    assert g.rank_exhausted and r.rank_exhausted
    assert g.rank == r.rank == 1
    assert_parity(g, r, o)


def test_stop_tol(ctx):
    x = wl.gen_c1(3000, 2, 5)
    g, r, o = run_both(x, "gaussian", 1.0, k=500, b=10, ctx=ctx, stop_tol=0.05)
    assert g.rank < 500
    assert g.relative_trace_error <= 0.05 + 1e-12
    assert_parity(g, r, o)


def test_tiny_n(ctx):
    x = np.array([[0.0], [1.0], [3.0]])
    g, r, o = run_both(x, "gaussian", 1.0, k=3, b=2, ctx=ctx)
    assert_parity(g, r, o)
    assert g.rank == 3


def test_reference_invariants_on_gpu_output(ctx):  # test_rpcholesky.cpp:226-355
    x = wl.gen_c2(3000, 20, 1)
    cfg = api.RunConfig.until_rank(100, 30, 4)
    g = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec("gaussian", 4.0)), cfg, ctx)
    assert len(set(g.pivots.tolist())) == g.rank
    u = g.residual_diag
    assert np.all(u >= 0.0) and np.all(u <= 1.0 + 1e-8)
    f = g.factor
    assert abs(u.sum() - (3000 - np.sum(f * f))) <= 1e-8 * 3000
    assert np.array_equal(g.chol_factor, np.tril(f[g.pivots]))
    assert abs(g.captured_sq - np.sum(f * f)) <= 1e-9 * 3000


def test_invalid_arguments(ctx):
    x = wl.gen_c1(100, 3, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", 1.0))
    with pytest.raises(ValueError, match="block size"):
        api.accelerated_rpcholesky(ko, api.RunConfig(block_size=0, target_rank=3), ctx)
    with pytest.raises(ValueError, match="bandwidth"):
        api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec("gaussian", -1.0)),
                                   api.RunConfig.until_rank(3, 2, 0), ctx)
    with pytest.raises(ValueError, match="GramTrick"):
        api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec("l1laplace", 1.0), "gram"),
                                   api.RunConfig.until_rank(3, 2, 0), ctx)
    bad = x.copy()
    bad[5, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        api.accelerated_rpcholesky(api.KernelOracle(bad, api.KernelSpec("gaussian", 1.0)),
                                   api.RunConfig.until_rank(3, 2, 0), ctx)


# --------------------------------------------------------------- sharding
@pytest.mark.parametrize("p", [2, 3, 5, 7])
def test_virtual_shards_p_invariance(p):  # p = 7: shards 5 and 6 own no rows
    x = wl.gen_c1(20000, 10, 0)
    cfg = api.RunConfig.until_rank(200, 40, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(10.0)))
    c1 = api.Context(0)
    cp = api.Context(0, virtual_shards=p)
    g1 = api.accelerated_rpcholesky(ko, cfg, c1)
    gp = api.accelerated_rpcholesky(ko, cfg, cp)
    assert np.array_equal(g1.pivots, gp.pivots)
    assert np.array_equal(g1.factor, gp.factor)          # bitwise
    assert g1.relative_trace_error == gp.relative_trace_error
    assert g1.captured_sq == gp.captured_sq
    assert np.array_equal(g1.chol_factor, gp.chol_factor)


# ------------------------------------------------------ streamed factor output
def test_factor_streamed_into_host_buffer(ctx):
    """rpc_accelerated_rpcholesky_into: the factor arrives in host memory during the rounds
    and is bitwise the device factor (rpc_result_factor_copy)."""
    w = wl.CONFIGS["C1"]
    ko = api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma))
    cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
    g = api.accelerated_rpcholesky_into(ko, cfg, None, ctx)          # pageable: registered
    ref = api.accelerated_rpcholesky(ko, cfg, ctx)
    assert np.array_equal(g.pivots, ref.pivots)
    assert np.array_equal(g.factor, ref.factor_into(np.zeros((w.n, ref.rank), order="F")))
    buf = np.zeros((w.n, api.factor_capacity(w.n, cfg) + 5), order="F")
    g2 = api.accelerated_rpcholesky_into(ko, cfg, buf, ctx)
    assert np.array_equal(g2.factor, g.factor)
    with pytest.raises(ValueError):
        api.accelerated_rpcholesky_into(ko, cfg, np.zeros((w.n, 3), order="F"), ctx)


@pytest.mark.parametrize("p", [3])
def test_factor_streamed_virtual_shards(p):
    x = wl.gen_c1(20000, 10, 0)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(10.0)))
    cfg = api.RunConfig.until_rank(200, 40, 0)
    a = api.accelerated_rpcholesky_into(ko, cfg, None, api.Context(0))
    b = api.accelerated_rpcholesky_into(ko, cfg, None, api.Context(0, virtual_shards=p))
    assert np.array_equal(a.factor, b.factor)


def test_bench_column_throughput_rows(ctx):
    """bench_column_throughput (experiment.hpp:344-387): one row per (block size, mode),
    ~1000 columns each, Direct + GramTrick for the Gaussian, Direct only for l1."""
    x = wl.gen_c2(30000, 12, 1)
    rows = api.bench_column_throughput(api.KernelOracle(x, api.KernelSpec("gaussian", 3.0)),
                                       [1, 7, 120, 300], 0, ctx)
    assert [(r["block_size"], r["mode"]) for r in rows] == [
        (1, "direct"), (1, "gram"), (7, "direct"), (7, "gram"), (120, "direct"), (120, "gram"),
        (300, "direct"), (300, "gram")]
    for r in rows:
        b = r["block_size"]
        assert r["columns"] == -(-1000 // b) * b
        assert r["wall_ms"] > 0 and r["columns_per_sec"] > 0
        assert abs(r["output_gbs"] - 8 * 30000 * r["columns"] / (r["wall_ms"] * 1e-3) / 1e9) < 1e-6 * r["output_gbs"]
    l1 = api.bench_column_throughput(api.KernelOracle(x, api.KernelSpec("l1laplace", 3.0)), [40],
                                     0, ctx)
    assert [r["mode"] for r in l1] == ["direct"]
    with pytest.raises(ValueError, match="block size"):
        api.bench_column_throughput(api.KernelOracle(x, api.KernelSpec("l1laplace", 3.0)), [0], 0, ctx)


@pytest.mark.parametrize("b,d,kernel", [(256, 8, "gaussian"), (256, 40, "l1laplace")])
def test_max_block_size(ctx, b, d, kernel):  # b = 256: the largest single-launch tile configuration
    x = wl.gen_c2(9000, d, 4)
    g, r, o = run_both(x, kernel, math.sqrt(d), k=600, b=b, ctx=ctx)
    assert_parity(g, r, o)


# b > 256 (rpcholesky.hpp:342 accepts any b >= 1): rounds whose accepted set exceeds 256 are
# appended in groups of 128 (block Cholesky against the sweep's L), the sweep holds H packed in
# L2; pivots must still equal the reference's and F agree to 1e-10
@pytest.mark.parametrize("b,d,kernel,replay", [(300, 8, "gaussian", False), (300, 8, "gaussian", True),
                                               (600, 20, "gaussian", False),
                                               (1024, 30, "l1laplace", False)])
def test_block_size_beyond_256(ctx, b, d, kernel, replay):
    x = wl.gen_c2(12000, d, 4)
    g, r, o = run_both(x, kernel, math.sqrt(d), k=2 * b, b=b, ctx=ctx, replay=replay)
    assert max(len(a) for a in g.accepted) > 128  # grouped appends really ran
    assert_parity(g, r, o)


def test_block_size_limits(ctx):
    x = wl.gen_c2(3000, 4, 4)
    with pytest.raises(ValueError, match="block size <= 1024"):
        api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec("gaussian", 1.0)),
                                   api.RunConfig.until_rank(10, 1025, 0), ctx)
    with pytest.raises(ValueError, match="block size <= 256"):
        api.accelerated_rpcholesky_lowmem(api.KernelOracle(x, api.KernelSpec("gaussian", 1.0)),
                                          api.RunConfig.until_rank(10, 257, 0), ctx)


@pytest.mark.parametrize("kernel,dist", [("matern32", None), ("matern32", "direct"),
                                         ("matern52", None), ("matern52", "direct")])
def test_matern_parity(ctx, kernel, dist):  # KernelKind::Matern32/52, kernels.hpp:66-75
    x = wl.gen_c2(6000, 8, 3)
    g, r, o = run_both(x, kernel, 2.5, k=250, b=60, ctx=ctx, dist=dist)
    assert_parity(g, r, o)


def test_nccl_context_single_rank():
    """rpc_create_nccl (the multi-GPU context) at world size 1 on this box: the NCCL
    communicator initialises and the factorization is bitwise the plain context's."""
    x = wl.gen_c1(6000, 8, 0)
    spec = api.KernelSpec("gaussian", math.sqrt(8.0))
    cfg = api.RunConfig.until_rank(60, 16, 5)
    plain = api.Context(0)
    ref = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, plain)
    f_ref = ref.factor.copy()
    plain.close()
    nc = api.Context(0, nccl_id=api.nccl_unique_id(), nranks=1, rank=0)
    got = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, nc)
    assert np.array_equal(got.pivots, ref.pivots)
    assert np.array_equal(got.factor, f_ref)
    nc.close()


# Dimensions around the 16-coordinate chunk and 4-wide k-step boundaries: the update
# kernel skips the zero padding of X (Gram k steps with no data, distance coordinates
# >= d), so every residue of d mod 16 and mod 4 must still give the reference's result.
@pytest.mark.parametrize("d", [1, 3, 4, 5, 15, 16, 17, 20, 31, 33, 47, 48])
@pytest.mark.parametrize("kernel,dist", [("gaussian", "gram"), ("gaussian", "direct"),
                                         ("l1laplace", None)])
def test_dimension_padding_boundaries(ctx, d, kernel, dist):
    rng = np.random.default_rng(100 + d)
    x = rng.standard_normal((3000, d))
    sigma = math.sqrt(d) if kernel == "gaussian" else float(d)
    # FixedRounds keeps the run bounded and, for the smooth kernel in very low d, inside the
    # kernel's numerical rank (past it both implementations factor rounding noise)
    rounds = 1 if (kernel == "gaussian" and d <= 3) else 3
    g, r, o = run_both(x, kernel, sigma, b=16, seed=d, rounds=rounds, ctx=ctx, dist=dist)
    assert_parity(g, r, o)


# Any d on the standard path (the reference's KernelOracle takes any dimension): the point pack
# stages fewer rows per CTA as d grows and takes a per-row kernel beyond the shared-memory
# tile; the Gram / distance phases stream X in 16-coordinate chunks.
@pytest.mark.parametrize("d,kernel,dist", [(500, "gaussian", None), (500, "l1laplace", None),
                                           (3300, "gaussian", "direct"), (30000, "gaussian", None)])
def test_large_dimension(ctx, d, kernel, dist):
    n = 3000 if d < 30000 else 600
    x = wl.gen_c3(n, d, 2)
    sigma = math.sqrt(d) * (0.5 if kernel == "gaussian" else 10.0)
    g, r, o = run_both(x, kernel, sigma, k=60, b=20, ctx=ctx, dist=dist)
    assert_parity(g, r, o)


# ------------------------------------------- fused sweep + round prep (one launch)
@pytest.mark.parametrize("n,d,b,k", [(20000, 10, 40, 200), (30000, 30, 120, 600), (8000, 3, 24, 96),
                                     (12000, 20, 128, 500), (6000, 5, 1, 20), (9000, 8, 17, 70)])
def test_fused_sweep_prep_bitwise_equals_two_launches(ctx, monkeypatch, n, d, b, k):
    """The fused launch (CTA 0 sweeps, the other warps form L^-1, B' and the operands behind
    its per-block progress word) must reproduce the two-launch path bit for bit: same
    pivots, and F, u, chol identical to the last bit (same operations per entry)."""
    x = wl.gen_c1(n, d, 3)
    spec = api.KernelSpec("gaussian", math.sqrt(d))
    cfg = api.RunConfig.until_rank(k, b, 11)
    monkeypatch.delenv("RPC_NO_FUSED_PREP", raising=False)
    a = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, ctx)
    monkeypatch.setenv("RPC_NO_FUSED_PREP", "1")
    r = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, ctx)
    assert np.array_equal(a.pivots, r.pivots)
    assert np.array_equal(a.factor, r.factor)
    assert np.array_equal(a.residual_diag, r.residual_diag)
    assert np.array_equal(a.chol_factor, r.chol_factor)
    assert a.relative_trace_error == r.relative_trace_error


def test_sample_from_thread_bases_equals_rescan(ctx, monkeypatch):
    """The sampler that reads the stored thread bases must pick exactly the rows the
    rescanning sampler picks (same fast cumsum), including zero plateaus, runs of zeros
    spanning whole 16-row runs and chunks, partial last chunks and the clamp case."""
    rng = np.random.default_rng(5)
    cases = []
    for n in (1, 17, 4096, 4097, 12289, 100000, 262144 + 7):
        u = rng.random(n) ** 4
        u[rng.random(n) < 0.3] = 0.0
        cases.append(u)
    u = rng.random(50000)
    u[:20000] = 0.0
    u[30000:] = 0.0          # trailing zero chunks: plateau walk back over whole chunks
    cases.append(u)
    u = np.zeros(9000)
    u[4095] = 1e-300         # a single tiny weight
    u[8191] = 2.0
    cases.append(u)
    for u in cases:
        if not np.any(u > 0):
            continue
        monkeypatch.delenv("RPC_NO_TB_SAMPLER", raising=False)
        a = api.sample_discrete(u, 300, 17, 5, replay=False, ctx=ctx)
        monkeypatch.setenv("RPC_NO_TB_SAMPLER", "1")
        b = api.sample_discrete(u, 300, 17, 5, replay=False, ctx=ctx)
        assert np.array_equal(a, b)
        assert np.all(u[a] > 0.0)


@pytest.mark.parametrize("n,d,b,k,shards", [(20000, 10, 40, 200, 1), (70000, 30, 120, 600, 1),
                                            (4097, 3, 24, 96, 1), (200000, 20, 128, 500, 1),
                                            (70000, 30, 120, 600, 3), (20000, 10, 40, 200, 2)])
def test_update_fused_scan_bitwise_equals_totals_pass(ctx, monkeypatch, n, d, b, k, shards):
    """Scan from the update's 16-row run sums (chunk chaining launch, thread-base sampler,
    offsets chained by the sampler on one shard or by the prefix pass across shards) against
    the totals pass over u: identical pivots and factor bit for bit."""
    x = wl.gen_c1(n, d, 4)
    spec = api.KernelSpec("gaussian", math.sqrt(d))
    cfg = api.RunConfig.until_rank(k, b, 13)
    c = ctx if shards == 1 else api.Context(0, virtual_shards=shards)
    monkeypatch.delenv("RPC_NO_FUSED_SCAN", raising=False)
    a = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, c)
    monkeypatch.setenv("RPC_NO_FUSED_SCAN", "1")
    r = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, c)
    assert np.array_equal(a.pivots, r.pivots)
    assert np.array_equal(a.factor, r.factor)
    assert np.array_equal(a.residual_diag, r.residual_diag)
    assert a.relative_trace_error == r.relative_trace_error
    if shards > 1:
        c.close()


@pytest.mark.parametrize("n,d,b,k,kernel", [(60000, 30, 120, 800, "gaussian"),
                                            (40000, 10, 64, 700, "gaussian"),
                                            (50000, 20, 100, 650, "laplace"),
                                            (40000, 24, 200, 900, "laplace"),
                                            (30000, 12, 300, 800, "gaussian")])
def test_tensor_core_residual_matches_dmma_and_oracle(ctx, monkeypatch, n, d, b, k, kernel):
    """Rounds past RPC_I8_MIN_K compute F B'^T from int8 digit planes on tcgen05 (i8gemm.cu):
    same pivots as the FP64 DMMA path and the oracle, factor within the parity bar.  b > 128:
    grouped rounds, each group's columns appended to the digit planes before the next group's
    product (the C5 shape)."""
    x = wl.gen_c1(n, d, 6)
    sigma = math.sqrt(d)
    spec = api.KernelSpec(kernel, sigma)
    cfg = api.RunConfig.until_rank(k, b, 21)
    monkeypatch.setenv("RPC_I8_MIN_K", "256")
    monkeypatch.delenv("RPC_NO_I8", raising=False)
    a = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, ctx)
    monkeypatch.setenv("RPC_NO_I8", "1")
    r = api.accelerated_rpcholesky(api.KernelOracle(x, spec), cfg, ctx)
    assert np.array_equal(a.pivots, r.pivots)
    rel = np.linalg.norm(a.factor - r.factor) / np.linalg.norm(r.factor)
    assert rel <= 1e-10, rel
    assert abs(a.relative_trace_error - r.relative_trace_error) <= 1e-12
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma, n_threads=8)
    ref = po.accelerated_rpcholesky(o, block_size=b, seed=21, target_rank=k)
    assert np.array_equal(a.pivots, ref.pivots)
    assert np.linalg.norm(a.factor - ref.factor) / np.linalg.norm(ref.factor) <= F_TOL
