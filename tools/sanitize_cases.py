"""Small runs of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Each case is checked against the CPU oracle so a sanitizer run also proves the results."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import pyoracle as po  # noqa: E402
from paper_2410_03969_b200 import api, workloads  # noqa: E402


def main():
    x = workloads.gen_c1(5000, 10, 0)
    sg = math.sqrt(10.0)
    ctx = api.Context(0)
    for kern, sigma, replay in (("gaussian", sg, False), ("gaussian", sg, True),
                                ("l1laplace", 3.0, False)):
        cfg = api.RunConfig.until_rank(80, 24, 0)
        cfg.replay_scan = replay
        g = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec(kern, sigma)), cfg, ctx)
        r = po.accelerated_rpcholesky(po.Oracle(x=x, kernel=kern, sigma=sigma, n_threads=8),
                                      block_size=24, target_rank=80, seed=0)
        assert np.array_equal(g.pivots, r.pivots), (kern, replay)
        rel = np.linalg.norm(g.factor - r.factor) / np.linalg.norm(r.factor)
        assert rel < 1e-10, rel
        g.free()
        print(f"accelerated {kern} replay={replay}: ok ({rel:.1e})")
    cfg = api.RunConfig.until_rank(80, 24, 0)
    lm = api.accelerated_rpcholesky_lowmem(api.KernelOracle(x, api.KernelSpec("gaussian", sg)), cfg, ctx)
    print("lowmem: ok", lm.rank)
    lm.free()
    bl = api.block_rpcholesky(api.KernelOracle(x, api.KernelSpec("gaussian", sg)), cfg, ctx)
    print("block: ok", bl.rank)
    bl.free()
    vctx = api.Context(0, virtual_shards=3)
    xv = workloads.gen_c1(10000, 10, 0)
    gv = api.accelerated_rpcholesky(api.KernelOracle(xv, api.KernelSpec("gaussian", sg)), cfg, vctx)
    g1 = api.accelerated_rpcholesky(api.KernelOracle(xv, api.KernelSpec("gaussian", sg)), cfg, ctx)
    assert np.array_equal(gv.factor, g1.factor)
    print("virtual shards: ok")
    gv.free()
    g1.free()
    vctx.close()
    cols = api.KernelOracle(x, api.KernelSpec("gaussian", sg)).columns([3, 17, 4000], ctx)
    print("columns: ok", cols.shape)
    t = np.sin(x[:, 0]) + 0.1 * x[:, 1]
    fit = api.fit_krr(x[:2000], t[:2000], api.KernelSpec("gaussian", sg), 1e-3, 100,
                      api.RunConfig.until_rank(100, 20, 0), 1e-8, 50, ctx)
    pred = api.predict(fit.model, x[2000:2100])
    print("krr: ok", fit.report.iterations, float(np.abs(pred).max()))
    fit.model.free()
    ctx.close()


if __name__ == "__main__":
    main()
