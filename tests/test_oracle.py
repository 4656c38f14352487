"""CPU oracle pinned against golden vectors and the reference's own test suites.

Ports the hot-path properties of
  /root/reference/proj/tests/test_rng.cpp
  /root/reference/proj/tests/test_kernel_oracle.cpp
  /root/reference/proj/tests/test_rpcholesky.cpp
onto the oracle restatement (oracle/rpc_oracle.c).  No GPU needed.
"""
import json
import math
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2410_03969_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def random_psd(n, r, seed):
    """test_support.hpp:23-33 (W filled column by column)."""
    w = wl.normals(seed, 0, n * r).reshape(r, n).T
    a = w @ w.T
    return 0.5 * (a + a.T)


def dense(a):
    return po.Oracle(dense=a)


def acc(oracle, **kw):
    return po.accelerated_rpcholesky(oracle, **kw)


# ---------------------------------------------------------------- rng.hpp
def test_splitmix64_golden_kat():
    kat = json.load(open(os.path.join(GOLDEN, "splitmix64_kat.json")))
    for seed, v in kat["seeds"].items():
        for n, (hx, dx) in enumerate(zip(v["u64_hex"], v["u01"])):
            z = po.splitmix64_draw(int(seed), n)
            assert z == int(hx, 16)
            assert po.u01(z) == float.fromhex(dx)
    for n, hx in kat["seed7_draw_n"].items():
        assert po.splitmix64_draw(7, int(n)) == int(hx, 16)


def test_splitmix64_numpy_counter_matches_oracle():
    z = wl.splitmix64_counter(42, 10, 50)
    assert [int(v) for v in z] == [po.splitmix64_draw(42, 10 + i) for i in range(50)]


def test_uniform_range():  # test_rng.cpp:23-34
    u = wl.uniforms(3, 0, 100000)
    assert u.min() >= 0.0 and u.max() < 1.0


def test_discrete_law_and_zero_weight():  # test_rng.cpp:49-73
    w = np.array([1.0, 0.0, 3.0, 0.0, 4.0])
    cs = po.cumulative_sums(w)
    counts = np.zeros(5)
    for t in range(40000):
        counts[po.sample_discrete(cs, po.u01(po.splitmix64_draw(11, t)))] += 1
    assert counts[1] == 0 and counts[3] == 0
    np.testing.assert_allclose(counts / counts.sum(), w / w.sum(), atol=0.01)


def test_discrete_all_zero_throws():  # test_rng.cpp:75-80
    with pytest.raises(ValueError):
        po.sample_discrete(po.cumulative_sums(np.zeros(4)), 0.5)
    with pytest.raises(ValueError):
        po.sample_discrete(np.zeros(0), 0.5)


def test_discrete_plateau_walk_and_clamp():  # rng.hpp:90-94
    cs = np.array([1.0, 2.0, 2.0, 2.0])
    # target = 1.0*total would be past the end -> clamp to n-1 -> walk back to 1
    assert po.sample_discrete(cs, 1.0) == 1
    assert po.sample_discrete(cs, 0.0) == 0
    assert po.sample_discrete(cs, 0.5) == 1   # target 1.0: first > 1.0 is index 1


def test_cumulative_sums_sequential_order():
    w = np.array([1e16, 1.0, 1.0, -1e16 + 4.0])
    w[3] = 1.0
    cs = po.cumulative_sums(w)
    acc_ = 0.0
    for i, v in enumerate(w):
        acc_ += v
        assert cs[i] == acc_


# ---------------------------------------------------------- kernels/oracle
def test_gaussian_half_pinned():  # test_kernel_oracle.cpp:37-40
    x = np.array([[0.0, 0.0], [1.0, 1.0]])
    o = po.Oracle(x=x, kernel="gaussian", sigma=1.0)
    assert o.submatrix([0], [1])[0, 0] == pytest.approx(math.exp(-1.0), rel=1e-15)


def test_l1_closed_form():  # test_kernel_oracle.cpp:41-47
    x = np.array([[0.0, 0.0], [1.0, 2.0]])
    o = po.Oracle(x=x, kernel="l1laplace", sigma=2.0)
    assert o.submatrix([0], [1])[0, 0] == pytest.approx(math.exp(-1.5), rel=1e-15)


@pytest.mark.parametrize("dist", ["gram", "direct"])
def test_345_both_modes(dist):  # test_kernel_oracle.cpp:107-112
    x = np.array([[0.0, 0.0], [3.0, 4.0]])
    o = po.Oracle(x=x, kernel="gaussian", sigma=5.0, dist=dist)
    assert o.submatrix([0], [1])[0, 0] == pytest.approx(math.exp(-0.5), rel=1e-14)


def test_same_index_exact_one():  # test_kernel_oracle.cpp:113-117
    x = wl.gen_c1(50, 7, 5) * 1e3   # large norms: Gram cancellation would bite
    o = po.Oracle(x=x, kernel="gaussian", sigma=0.3)
    idx = np.arange(50)
    h = o.submatrix(idx, idx)
    assert np.all(np.diag(h) == 1.0)


def test_gram_matches_direct():  # test_kernel_oracle.cpp:126-139, 183-210
    x = wl.gen_c1(300, 6, 9)
    g = po.Oracle(x=x, kernel="gaussian", sigma=1.7, dist="gram")
    d = po.Oracle(x=x, kernel="gaussian", sigma=1.7, dist="direct")
    r, c = np.arange(300), np.arange(0, 300, 7)
    assert np.max(np.abs(g.submatrix(r, c) - d.submatrix(r, c))) <= 1e-10


def test_identical_points_all_ones():  # test_kernel_oracle.cpp:143-149
    x = np.tile(np.array([[0.3, -1.2, 2.0]]), (5, 1))
    for kern in ("gaussian", "l1laplace"):
        o = po.Oracle(x=x, kernel=kern, sigma=0.5)
        assert np.all(o.submatrix(np.arange(5), np.arange(5)) == 1.0)


@pytest.mark.parametrize("kern", ["gaussian", "l1laplace"])
def test_symmetric_psd_and_transpose(kern):  # test_kernel_oracle.cpp:168-181, 225-233
    x = wl.gen_c3(60, 4, 2)
    o = po.Oracle(x=x, kernel=kern, sigma=0.8)
    a = o.submatrix(np.arange(60), np.arange(60))
    assert np.max(np.abs(a - a.T)) < 1e-14
    assert np.linalg.eigvalsh(a).min() >= -1e-10 * np.trace(a)


def test_diag_equals_1x1_blocks():  # test_kernel_oracle.cpp:212-223
    x = wl.gen_c1(40, 3, 1)
    o = po.Oracle(x=x, kernel="gaussian", sigma=2.0)
    for i in range(40):
        assert o.submatrix([i], [i])[0, 0] == 1.0


def test_thread_count_bit_identity():  # test_kernel_oracle.cpp:235-248
    x = wl.gen_c1(700, 5, 4)
    cols = np.arange(0, 700, 1)[:600]
    a1 = po.Oracle(x=x, kernel="gaussian", sigma=1.0, n_threads=1).submatrix(np.arange(700), cols)
    a4 = po.Oracle(x=x, kernel="gaussian", sigma=1.0, n_threads=4).submatrix(np.arange(700), cols)
    assert np.array_equal(a1, a4)


def test_gram_rejected_for_l1_and_bad_inputs():  # test_kernel_oracle.cpp:250-256
    x = np.zeros((3, 2))
    with pytest.raises(ValueError):
        po.Oracle(x=x, kernel="l1laplace", sigma=1.0, dist="gram")
    with pytest.raises(ValueError):
        po.Oracle(x=x, kernel="gaussian", sigma=0.0)
    with pytest.raises(ValueError):
        po.Oracle(x=np.array([[np.nan, 1.0]]), kernel="gaussian", sigma=1.0)
    o = po.Oracle(x=x, kernel="gaussian", sigma=1.0)
    with pytest.raises(IndexError):
        o.submatrix([3], [0])


# ------------------------------------------------------------- rpcholesky
def test_sweep_single_proposal_always_accepted():  # test_rpcholesky.cpp:98-110
    for seed in range(200):
        acc_ids, pos, L = po.rejection_sweep(np.array([[0.37]]), [5], seed, 0)
        assert list(acc_ids) == [5]
        assert L[0, 0] == pytest.approx(math.sqrt(0.37))


def test_sweep_duplicate_never_twice():  # test_rpcholesky.cpp:111-120
    h = np.full((2, 2), 2.0)
    for seed in range(3000):
        acc_ids, _, _ = po.rejection_sweep(h, [3, 3], seed, 0)
        assert len(acc_ids) == 1


def test_sweep_diagonal_accepts_all():  # test_rpcholesky.cpp:121-129
    h = np.diag([0.5, 1.5, 0.25])
    for seed in range(500):
        assert len(po.rejection_sweep(h, [0, 1, 2], seed, 0)[0]) == 3


def test_accelerated_b1_accepts_everything():  # test_rpcholesky.cpp:187-197
    a = random_psd(20, 20, 6) + 0.2 * np.eye(20)
    res = acc(dense(a), block_size=1, mode="fixed_rounds", rounds=15, seed=101)
    assert all(len(r) == 1 for r in res.accepted)
    assert res.rank == 15


def test_exact_rank_termination():  # test_rpcholesky.cpp:199-212
    for r in range(1, 5):
        a = random_psd(16, r, 70 + r)
        o = dense(a)
        res = acc(o, block_size=2, target_rank=r, seed=55 + r)
        assert po.relative_trace_error(o, res.factor) <= 1e-9


def test_first_proposal_always_accepted():  # test_rpcholesky.cpp:214-224
    o = dense(random_psd(24, 24, 8))
    for seed in range(20):
        res = acc(o, block_size=4, mode="fixed_rounds", rounds=5, seed=seed)
        assert all(len(r) >= 1 for r in res.accepted)


def test_distinct_pivots():  # test_rpcholesky.cpp:226-235
    o = dense(random_psd(12, 12, 9))
    for seed in range(30):
        res = acc(o, block_size=3, target_rank=10, seed=seed)
        assert len(set(res.pivots.tolist())) == len(res.pivots)


def test_until_rank_surplus():  # test_rpcholesky.cpp:237-252
    o = dense(random_psd(40, 40, 10) + 0.5 * np.eye(40))
    saw = False
    for seed in range(40):
        res = acc(o, block_size=4, target_rank=9, seed=seed)
        assert res.rank >= 9
        if res.rank > 9:
            saw = True
            assert res.surplus == res.rank - 9
            break
    assert saw


@pytest.mark.parametrize("rep", range(4))
def test_psd_residual_trace_identity_interpolation(rep):  # test_rpcholesky.cpp:309-343
    a = random_psd(24, 24, 14 + rep)
    o = dense(a)
    tr = np.trace(a)
    res = acc(o, block_size=3, target_rank=10, seed=500 + rep)
    f = res.factor
    resid = a - f @ f.T
    assert np.linalg.eigvalsh(0.5 * (resid + resid.T)).min() >= -1e-8 * tr
    assert abs(np.trace(resid) - (tr - np.sum(f * f))) <= 1e-9 * tr
    for s in res.pivots:
        assert abs(resid[s, s]) <= 1e-8 * tr
    ass = a[np.ix_(res.pivots, res.pivots)]
    assert np.max(np.abs(res.chol @ res.chol.T - ass)) <= 1e-8 * tr


def test_residual_diag_invariants():  # test_rpcholesky.cpp:345-355
    a = random_psd(20, 20, 15)
    o = dense(a)
    tr = np.trace(a)
    for seed in range(10):
        res = acc(o, block_size=4, target_rank=8, seed=seed)
        assert np.all(res.residual_diag >= 0.0)
        assert np.all(res.residual_diag - np.diag(a) <= 1e-8 * tr)


def test_prefix_property_monotone_error():  # test_rpcholesky.cpp:357-372
    a = random_psd(24, 24, 16)
    o = dense(a)
    for seed in range(5):
        last, prev = 1.0, None
        for t in range(1, 7):
            res = acc(o, block_size=3, mode="fixed_rounds", rounds=t, seed=seed)
            err = po.relative_trace_error(o, res.factor)
            assert err <= last + 1e-10
            last = err
            if prev is not None:  # fewer rounds is a prefix of more rounds
                assert np.array_equal(res.pivots[: len(prev)], prev)
            prev = res.pivots


def test_stream_layout_replay():  # test_rpcholesky.cpp:374-404
    a = random_psd(12, 12, 18)
    o = dense(a)
    b, seed = 4, 4242
    res = acc(o, block_size=b, mode="fixed_rounds", rounds=2, seed=seed)
    u = np.diag(a).copy()
    cs = po.cumulative_sums(u)
    prop = [po.sample_discrete(cs, po.u01(po.splitmix64_draw(seed, j))) for j in range(b)]
    assert np.array_equal(prop, res.proposed[0])
    h = o.submatrix(prop, prop)
    acc_ids, _, L = po.rejection_sweep(h, prop, seed, b)
    assert np.array_equal(acc_ids, res.accepted[0])
    g = o.columns(acc_ids)
    g = np.linalg.solve(L, g.T).T
    u = np.maximum(u - np.sum(g * g, axis=1), 0.0)
    cs = po.cumulative_sums(u)
    prop2 = [po.sample_discrete(cs, po.u01(po.splitmix64_draw(seed, 2 * b + j))) for j in range(b)]
    assert np.array_equal(prop2, res.proposed[1])


def test_stop_tol():  # test_rpcholesky.cpp:406-415
    o = dense(random_psd(30, 30, 17))
    res = acc(o, block_size=5, target_rank=30, seed=9, stop_tol=0.2)
    assert po.relative_trace_error(o, res.factor) <= 0.2
    assert res.rank < 30


def test_invalid_config():  # rpcholesky.hpp:342-345
    o = dense(np.eye(3))
    with pytest.raises(ValueError):
        acc(o, block_size=0, target_rank=2)
    with pytest.raises(ValueError):
        acc(dense(np.zeros((3, 3))), block_size=1, target_rank=2)


def test_kernel_run_small_c1_like_properties():
    x = wl.gen_c1(3000, 10, 0)
    o = po.Oracle(x=x, kernel="gaussian", sigma=math.sqrt(10.0))
    res = acc(o, block_size=40, target_rank=200, seed=0)
    assert res.rank >= 200
    assert len(set(res.pivots.tolist())) == res.rank
    err = po.relative_trace_error(o, res.factor)
    assert 0.0 <= err < 1.0
    # trace identity through the residual diagonal: sum(u) ~ N - ||F||^2
    assert abs(res.residual_diag.sum() - (3000 - np.sum(res.factor ** 2))) <= 1e-8 * 3000
    # chol factor equals the pivot rows of F (lower part)
    assert np.array_equal(res.chol, np.tril(res.factor[res.pivots]))
