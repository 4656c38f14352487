"""Two ranks through librpchol_b200's own multi-rank path, on one B200.

Each rank is a separate process with its own context created by rpc_create_hostcoll: the
library runs the real sharded protocol (chunk-total allgather, owner-resolved draws,
proposal-record owner reduce, replicated H block / sweep / L^{-1}, rank-local fused
update, ||G||^2 allgather, chol owner reduce) and only the transport is the host
(torch.distributed over gloo, paper_2410_03969_b200/hostcoll.py) instead of NCCL.  The
kernels of one rank never wait on the other's, so sharing a GPU is safe.

Each rank's rows of the factor, its residual diagonal, the pivots, the PivotTrace and
chol_factor must be bitwise equal to a 1-rank run (p-invariance), for the
fast and the replay scan, the low-memory variant and block RPCholesky; write_rpcf from two
ranks must produce the same bytes as from one.
"""
import math
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_2410_03969_b200 import workloads as wl

pytestmark = pytest.mark.gpu

N, D = 30_000, 10          # 8 scan chunks: rank 0 owns rows [0, 16384), rank 1 the rest
SIGMA = math.sqrt(10.0)


def _cases():
    return {
        "fast": dict(algo="accelerated", replay=False),
        "replay": dict(algo="accelerated", replay=True),
        "lowmem": dict(algo="lowmem", replay=False),
        "block": dict(algo="block", replay=False),
        "l1_fixed": dict(algo="accelerated", replay=True, kernel="l1laplace", rounds=4),
    }


def _run(ctx, x, case, rpcf=None):
    from paper_2410_03969_b200 import api
    kern = case.get("kernel", "gaussian")
    sigma = SIGMA if kern == "gaussian" else 5.0
    cfg = (api.RunConfig.fixed_rounds(case["rounds"], 40, 0) if "rounds" in case
           else api.RunConfig.until_rank(200, 40, 0))
    cfg.replay_scan = case["replay"]
    ko = api.KernelOracle(x, api.KernelSpec(kern, sigma))
    fn = {"accelerated": api.accelerated_rpcholesky, "lowmem": api.accelerated_rpcholesky_lowmem,
          "block": api.block_rpcholesky}[case["algo"]]
    r = fn(ko, cfg, ctx)
    out = {"pivots": r.pivots, "proposed": np.array(r.proposed),
           "acc_counts": np.array([len(a) for a in r.accepted]),
           "chol": r.chol_factor, "resid": r.residual_diag,
           "err": np.array([r.relative_trace_error]), "surplus": np.array([r.surplus])}
    if case["algo"] != "lowmem":
        out["factor"] = r.factor
        if rpcf:
            r.write_rpcf(rpcf)
    r.free()
    if case["algo"] == "accelerated" and not case["replay"]:
        # the streamed-factor entry (rpc_accelerated_rpcholesky_into): each rank's rows land in
        # a full-height host buffer while the rounds run
        ri = api.accelerated_rpcholesky_into(ko, cfg, ctx=ctx)
        out["factor_into"] = np.array(ri.factor)
        ri.free()
    return out


def _worker(rank, port, tmp, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        from paper_2410_03969_b200 import api
        from paper_2410_03969_b200.hostcoll import TorchHostCollectives
        dist.init_process_group("gloo", rank=rank, world_size=2)
        ctx = api.Context(0, host_collectives=TorchHostCollectives())
        x = wl.gen_c1(N, D, 0)
        for name, case in _cases().items():
            rpcf = os.path.join(tmp, f"two_{name}.rpcf") if name == "fast" else None
            np.savez(os.path.join(tmp, f"rank{rank}_{name}.npz"), **_run(ctx, x, case, rpcf))
        # a non-finite entry on rank 1's rows is reported on both ranks
        xb = x.copy()
        xb[N - 5, 3] = np.nan
        try:
            _run(ctx, xb, _cases()["fast"])
            errq.put((rank, "no error"))
        except ValueError as e:
            assert "non-finite" in str(e)
        r0, nr = ctx.shard_rows(N)
        np.save(os.path.join(tmp, f"rows{rank}.npy"), np.array([r0, nr]))
        ctx.close()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        errq.put((rank, repr(e)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def two_rank_outputs(tmp_path_factory):
    tmp = str(tmp_path_factory.mktemp("two_rank"))
    ctxm = mp.get_context("spawn")
    errq = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, port, tmp, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs) and not errs, errs
    return tmp


@pytest.mark.parametrize("name", list(_cases()))
def test_two_ranks_bitwise_equal_one_rank(two_rank_outputs, name):
    from paper_2410_03969_b200 import api
    tmp = two_rank_outputs
    x = wl.gen_c1(N, D, 0)
    ctx = api.Context(0)
    one = _run(ctx, x, _cases()[name],
               os.path.join(tmp, f"one_{name}.rpcf") if name == "fast" else None)
    ctx.close()
    for rank in range(2):
        two = np.load(os.path.join(tmp, f"rank{rank}_{name}.npz"))
        r0, nr = np.load(os.path.join(tmp, f"rows{rank}.npy"))
        assert nr > 0
        for key in ("pivots", "proposed", "acc_counts", "chol", "err", "surplus"):
            assert np.array_equal(two[key], one[key]), (rank, key)
        assert np.array_equal(two["resid"][r0:r0 + nr], one["resid"][r0:r0 + nr]), rank
        if "factor" in one:
            assert np.array_equal(two["factor"][r0:r0 + nr], one["factor"][r0:r0 + nr]), rank
        if "factor_into" in one:
            assert np.array_equal(one["factor_into"], one["factor"])
            assert np.array_equal(two["factor_into"][r0:r0 + nr], one["factor"][r0:r0 + nr]), rank
    if name == "fast":
        with open(os.path.join(tmp, "two_fast.rpcf"), "rb") as a, \
                open(os.path.join(tmp, "one_fast.rpcf"), "rb") as b:
            assert a.read() == b.read()
