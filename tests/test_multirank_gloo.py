"""Multi-rank (N > 1) path on CPU with torch.distributed/gloo, world_size 2.

The B200 library shards rows over GPUs with the host plan of the C-ABI
(rpc_plan_shards) and exchanges, per round, only chunk totals and the owners'
proposal records.  Here two gloo ranks run that protocol around the CPU mirror of
the GPU sampler (oracle/chunkscan.py) and must reproduce the single-process result
exactly; the GPU test checks the CUDA sampler against the same mirror bit for bit.
The last test runs the whole row-sharded factorization protocol (records allgather,
replicated H block and sweep, rank-local update) at world size 1 and 2 against the
reference restatement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import chunkscan as cs
import pyoracle as po


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_u(n, seed):
    rng = np.random.default_rng(seed)
    u = rng.random(n) ** 2
    u[rng.random(n) < 0.25] = 0.0
    u[-1000:] = 0.0          # trailing plateau exercises the clamp walk
    return u


def _rank_main(rank, world, port, n, seed, b, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_03969_b200 import api
    plan = api.plan_shards(n, world, rank)
    u = make_u(n, seed)
    u_loc = [float(v) for v in u[plan["row0"]: plan["row0"] + plan["nrows"]]]
    # 1. chunk totals of the own shard, padded to chunks_per_shard, allgathered
    cpr = plan["chunks_per_shard"]
    tot = cs.chunk_totals(u_loc) + [0.0] * (cpr - plan["nchunks"])
    buf = [torch.zeros(cpr, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(buf, torch.tensor(tot, dtype=torch.float64))
    totals = [float(v) for t in buf for v in t.tolist()]
    ends = cs.chunk_ends(totals)
    # 2. every rank locates every draw; the owner resolves it; allgather of proposals
    mine = []
    for j in range(b):
        c, mode, target = cs.locate(ends, cs.u01(cs.splitmix64_draw(seed, j)))
        owner = c // cpr
        if owner == rank:
            lc = c - plan["chunk0"]
            off = ends[c - 1] if c else 0.0
            i = cs.resolve(u_loc[lc * cs.KCHUNK:(lc + 1) * cs.KCHUNK], off, mode, target)
            mine.append(plan["row0"] + lc * cs.KCHUNK + i)
        else:
            mine.append(-1)
    got = [torch.zeros(b, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, torch.tensor(mine, dtype=torch.int64))
    merged = torch.stack(got).max(dim=0).values.tolist()
    if rank == 0:
        out_q.put(merged)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [9000, 20000])
def test_two_rank_protocol_matches_single_process(n):
    seed, b = 7, 48
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, n, seed, b, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert merged == cs.sample(make_u(n, seed), seed, 0, b)


def test_plan_is_chunk_aligned_and_p_invariant():
    from paper_2410_03969_b200 import api
    for n in (1, 4095, 4096, 4097, 20000, 1_000_000):
        for P in (1, 2, 3, 8):
            plans = [api.plan_shards(n, P, s) for s in range(P)]
            assert plans[0]["row0"] == 0
            for a, bb in zip(plans, plans[1:]):
                assert a["row0"] + a["nrows"] == bb["row0"]
            assert plans[-1]["row0"] + plans[-1]["nrows"] == n
            for p in plans:
                assert p["row0"] % cs.KCHUNK == 0 or p["nrows"] == 0
                assert p["chunk0"] * cs.KCHUNK == p["row0"] or p["nrows"] == 0
    with pytest.raises(ValueError):
        api.plan_shards(10, 2, 2)


def test_fast_sampler_mirror_agrees_with_reference_sequential():
    # same draws, sequential cumsum (reference) vs fixed two-level order (GPU fast mode)
    for n, seed in ((5000, 1), (30000, 2)):
        u = make_u(n, seed)
        want = [po.sample_discrete(po.cumulative_sums(u), cs.u01(cs.splitmix64_draw(seed, j)))
                for j in range(200)]
        assert cs.sample(u, seed, 0, 200) == want


@pytest.mark.gpu
def test_gpu_fast_sampler_bit_exact_vs_mirror():
    from paper_2410_03969_b200 import api
    for n, seed in ((5000, 3), (12289, 4), (40000, 5)):
        u = make_u(n, seed)
        got = api.sample_discrete(u, 100, seed, 0, replay=False)
        assert list(got) == cs.sample(u, seed, 0, 100)


# ---- the whole row-sharded factorization over gloo ------------------------------------
# Each rank owns its chunk-aligned rows of X, F and u (rpc_plan_shards) and runs the B200
# library's per-round protocol (api.cu run_factorization) with the CPU oracle as the
# arithmetic: allgather of chunk totals -> every rank locates every draw, the owner
# resolves it and contributes the proposal record (id + F row) -> allgather of records
# -> H block and rejection sweep replicated on every rank -> rank-local update of its
# rows -> allgather of the per-rank ||G||^2.  World size 2 must reproduce world size 1
# and the reference's accelerated_rpcholesky (pivots identical, F to 1e-10).

def _sharded_run(rank, world, x, kernel, sigma, k, b, seed, comm):
    from scipy.linalg import solve_triangular
    from paper_2410_03969_b200 import api
    n = x.shape[0]
    o = po.Oracle(x=x, kernel=kernel, sigma=sigma)   # kernel values only (op order of the reference)
    plan = api.plan_shards(n, world, rank)
    r0, nl, cpr = plan["row0"], plan["nrows"], plan["chunks_per_shard"]
    rows = np.arange(r0, r0 + nl, dtype=np.int64)
    cap = min(n, k + b)
    f_loc = np.zeros((nl, cap))
    u_loc = np.ones(nl)                   # diag(A) = 1 for the kernel oracles (oracle.hpp:263)
    kcur, pivots, proposed, accepted, captured = 0, [], [], [], 0.0
    rnd = 0
    while kcur < k:
        draw0 = 2 * b * rnd
        tot = cs.chunk_totals([float(v) for v in u_loc]) + [0.0] * (cpr - plan["nchunks"])
        totals = [v for t in comm(np.array(tot)) for v in t]
        ends = cs.chunk_ends(totals)
        if not ends[-1] > 0.0:
            break                           # rank exhausted (rpcholesky.hpp:356-359)
        rec = np.zeros((b, 1 + cap))
        for j in range(b):
            c, mode, target = cs.locate(ends, cs.u01(cs.splitmix64_draw(seed, draw0 + j)))
            if c // cpr != rank:
                continue
            lc = c - plan["chunk0"]
            off = ends[c - 1] if c else 0.0
            i = lc * cs.KCHUNK + cs.resolve([float(v) for v in u_loc[lc * cs.KCHUNK:(lc + 1) * cs.KCHUNK]],
                                            off, mode, target)
            rec[j, 0] = r0 + i
            rec[j, 1:] = f_loc[i]
        rec = np.sum(comm(rec), axis=0)     # each slot has exactly one owner
        prop = rec[:, 0].astype(np.int64)
        fsp = rec[:, 1:1 + kcur]
        h = o.submatrix(prop, prop) - fsp @ fsp.T
        acc, pos, lmat = po.rejection_sweep(h, prop, seed, draw0 + b)
        m = len(acc)
        if m:
            g = o.submatrix(rows, acc) - f_loc[:, :kcur] @ fsp[pos].T
            g = solve_triangular(lmat, g.T, lower=True).T
            f_loc[:, kcur:kcur + m] = g
            u_loc = np.maximum(u_loc - np.sum(g * g, axis=1), 0.0)
            captured += float(np.sum(comm(np.array([np.sum(g * g)]))))
            pivots += [int(v) for v in acc]
            kcur += m
        proposed.append(prop)
        accepted.append(np.asarray(acc, np.int64))
        rnd += 1
    return dict(pivots=pivots, f=f_loc[:, :kcur], u=u_loc, proposed=proposed, accepted=accepted,
                captured=captured, row0=r0)


def _factor_rank_main(rank, world, port, args, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def comm(a):
        a = torch.as_tensor(np.asarray(a, dtype=np.float64))
        out = [torch.zeros_like(a) for _ in range(world)]
        dist.all_gather(out, a)
        return [t.numpy() for t in out]

    r = _sharded_run(rank, world, *args, comm)
    out_q.put((rank, r))
    dist.destroy_process_group()


def _run_world(world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_factor_rank_main, args=(r, world, port, args, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = np.vstack([parts[r]["f"] for r in range(world)])
    u = np.concatenate([parts[r]["u"] for r in range(world)])
    return parts[0], f, u


@pytest.mark.parametrize("kernel,sigma", [("gaussian", 1.5), ("l1laplace", 2.0)])
def test_two_rank_factorization_matches_one_rank_and_reference(kernel, sigma):
    n, d, k, b, seed = 9000, 5, 48, 16, 3
    rng = np.random.default_rng(11)
    x = rng.standard_normal((n, d))
    args = (x, kernel, sigma, k, b, seed)
    one, f1, u1 = _run_world(1, args)
    two, f2, u2 = _run_world(2, args)
    # the protocol is p-invariant: same proposals, decisions and factor
    assert [list(p) for p in one["proposed"]] == [list(p) for p in two["proposed"]]
    assert one["pivots"] == two["pivots"] and len(one["pivots"]) >= k
    assert np.linalg.norm(f1 - f2) <= 1e-12 * np.linalg.norm(f1)
    assert np.max(np.abs(u1 - u2)) <= 1e-12
    assert abs(one["captured"] - two["captured"]) <= 1e-10 * one["captured"]
    # and it is the reference's algorithm (rpc_oracle restatement of rpcholesky.hpp:338-401)
    ref = po.accelerated_rpcholesky(po.Oracle(x=x, kernel=kernel, sigma=sigma), block_size=b,
                                    target_rank=k, seed=seed)
    assert list(ref.pivots) == two["pivots"]
    assert [list(a) for a in ref.accepted] == [list(a) for a in two["accepted"]]
    assert np.linalg.norm(ref.factor - f2) <= 1e-10 * np.linalg.norm(ref.factor)
    assert np.max(np.abs(ref.residual_diag - u2)) <= 1e-10


def _hostcoll_main(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2410_03969_b200.hostcoll import TorchHostCollectives
    hc = TorchHostCollectives()
    send = np.arange(10, dtype=np.uint8) + 16 * rank
    gathered = hc.allgather(send)
    # owner reduce: rank r owns words r, r+2, ...; negative doubles, -0.0 and NaN payloads
    # must come back bit for bit (the library reduces fp64 records this way)
    vals = np.array([-1.5, -0.0, np.nan, 3.25, -np.inf, 1e-310], dtype=np.float64)
    buf = np.zeros(vals.size, dtype=np.uint64)
    own = np.arange(vals.size) % world == rank
    buf[own] = vals.view(np.uint64)[own]
    hc.allreduce_or(buf)
    out_q.put((rank, gathered.tolist(), buf.tolist()))
    dist.destroy_process_group()


def test_host_collectives_adapter_two_ranks():
    """paper_2410_03969_b200/hostcoll.py, the transport of rpc_create_hostcoll, at world 2."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_hostcoll_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    vals = np.array([-1.5, -0.0, np.nan, 3.25, -np.inf, 1e-310], dtype=np.float64)
    for rank, gathered, buf in res:
        assert gathered == list(range(10)) + list(range(16, 26))
        assert np.array_equal(np.array(buf, dtype=np.uint64), vals.view(np.uint64))
