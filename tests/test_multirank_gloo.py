"""Multi-rank (N > 1) path on CPU with torch.distributed/gloo, world_size 2.

The B200 library shards rows over GPUs with the host plan of the C-ABI
(rpc_plan_shards) and exchanges, per round, only chunk totals and the owners'
proposal records.  Here two gloo ranks run that protocol around the CPU mirror of
the GPU sampler (oracle/chunkscan.py) and must reproduce the single-process result
exactly; the GPU test checks the CUDA sampler against the same mirror bit for bit.
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
