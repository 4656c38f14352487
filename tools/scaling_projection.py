"""Measured one-GPU phase split of C4 and the row-sharded projection to P GPUs.

With P virtual shards on one B200 (rpc_create_virtual), every shard's fused update launch
processes exactly the rows one GPU of a P-GPU job would (same kernel, same sizes), so the
per-GPU update time at P is measured here directly (sum over the shards' launches / P; the
shards are chunk-aligned and equal but for the last).  The replicated per-round chain
(chunk totals, sampler, H block, sweep, round prep) runs on every GPU at full size: it is
taken from the P = 1 run.  The update (FP64 fused kernel + tensor-core residual) and the
digit-plane appends are row-local: their sum over the shards / P is one GPU's share.  The exchange per round (chunk-total allgather, record owner
reduce, ||G||^2 allgather) is not measurable on one GPU; it is charged at a stated estimate
per collective (--coll-us, default 15 us: small NCCL collectives over NVLink/NVSwitch).

  python tools/scaling_projection.py [--coll-us 15] > profiles/r02_scaling_projection.json

The conservative columns take the chain from the P-shard run itself (fact - update there):
the sharded scan path (per-shard totals, allgather, prefix) with every shard's small launches
serialised on the one GPU, so it over-states what P GPUs would pay.
"""
import argparse
import json
import os

# phases are measured serialised: the digit-plane appends stay on the main stream here (the
# library overlaps them with the next round's chain; that overlap is not credited below)
os.environ["RPC_NO_AUX_SLICE"] = "1"
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2410_03969_b200 import _lib as L  # noqa: E402
from paper_2410_03969_b200 import api, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--coll-us", type=float, default=15.0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    w = workloads.CONFIGS[args.config]
    x = np.ascontiguousarray(w.points())
    xd = torch.from_numpy(x).cuda()
    spec = api.KernelSpec(w.kernel, w.sigma)
    cfg = api.RunConfig.until_rank(w.k, w.b, w.seed)
    out = {"config": args.config, "coll_us_estimate": args.coll_us,
           "note": "RPC_NO_AUX_SLICE=1: appends serialised with the chain (overlap not credited)",
           "rows": []}
    base = None
    for P in (1, 2, 4, 8):
        ctx = api.Context(0, virtual_shards=P)
        t_fact, t_upd, t_sl, rounds, piv = [], [], [], 0, None
        for i in range(args.reps + 1):
            r = api.accelerated_rpcholesky_device(xd.data_ptr(), w.n, w.d, w.d, L.RPC_ROW_MAJOR,
                                                  spec, cfg, ctx)
            if i:
                t_fact.append(r.timing["factorize_ms"])
                t_upd.append(r.timing["update_ms"])
                t_sl.append(r.timing["tc_slice_ms"])  # digit-plane appends: per-shard work
            rounds, piv = len(r.proposed), r.pivots.copy()
            r.free()
        ctx.close()
        fact, upd = statistics.median(t_fact), statistics.median(t_upd)
        upd += statistics.median(t_sl)  # (row-local like the update)
        if base is None:
            base = {"factorize_ms": fact, "update_ms": upd, "chain_ms": fact - upd, "pivots": piv}
        per_gpu_update = upd / P
        colls = 0 if P == 1 else 3 * rounds  # chunk totals (+ g2) allgathers, record reduce
        proj = per_gpu_update + base["chain_ms"] + colls * args.coll_us * 1e-3
        # conservative: the chain as the P-shard run measures it (the sharded scan path, every
        # shard's small launches serialised on the one GPU, device-local exchange)
        chain_p = fact - upd
        proj_c = per_gpu_update + chain_p + colls * args.coll_us * 1e-3
        out["rows"].append({
            "P": P, "virtual_run_factorize_ms": fact, "update_ms_all_shards": upd,
            "per_gpu_update_ms": per_gpu_update, "replicated_chain_ms": base["chain_ms"],
            "collectives": colls, "projected_ms": proj,
            "projected_speedup": base["factorize_ms"] / proj,
            "chain_ms_sharded_run": chain_p, "projected_ms_conservative": proj_c,
            "projected_speedup_conservative": base["factorize_ms"] / proj_c,
            "pivots_equal_to_P1": bool(np.array_equal(piv, base["pivots"]))})
    out["rounds"] = rounds
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
