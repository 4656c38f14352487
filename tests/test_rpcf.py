"""RPCF factor file and pivot-trace CSV (io.hpp:218-293, 336-350).

Pins: oracle/pyoracle.write_rpcf / write_pivot_trace_csv produce files byte-identical to the
reference's own write_rpcf / write_pivot_trace_csv for the same run (oracle/_ref), and
read_rpcf round-trips.  The GPU writer (rpc_result_write_rpcf) streams the device factor
through pinned double buffers: its file must be byte-identical to the restatement's file
for the GPU's own factor, pivots and chol_factor (the bytes are the device values), must
read back through the reference's read_rpcf, and must not depend on the shard count.
"""
import math
import os

import numpy as np
import pytest

import pyoracle as po
import pyref
from paper_2410_03969_b200 import workloads as wl


@pytest.mark.skipif(not pyref.available(), reason="oracle/_ref not built")
def test_restatement_writes_reference_bytes(tmp_path):
    x = wl.gen_c1(3000, 10, 0)
    pyref.write_rpcf_kernel(x, "gaussian", math.sqrt(10), 40, 200, 0, str(tmp_path / "ref.rpcf"),
                            str(tmp_path / "ref.csv"))
    o = po.Oracle(x=x, kernel="gaussian", sigma=math.sqrt(10))
    r = po.accelerated_rpcholesky(o, block_size=40, target_rank=200)
    po.write_rpcf(str(tmp_path / "po.rpcf"), r.factor, r.pivots, r.chol)
    po.write_pivot_trace_csv(str(tmp_path / "po.csv"), r.proposed, r.accepted)
    assert (tmp_path / "ref.rpcf").read_bytes() == (tmp_path / "po.rpcf").read_bytes()
    assert (tmp_path / "ref.csv").read_text() == (tmp_path / "po.csv").read_text()
    f, p, c = pyref.read_rpcf(str(tmp_path / "po.rpcf"))
    assert np.array_equal(f, r.factor) and np.array_equal(p, r.pivots) and np.array_equal(c, r.chol)


def test_restatement_roundtrip_and_edge_cases(tmp_path):
    rng = np.random.default_rng(0)
    f = rng.standard_normal((37, 5))
    c = np.tril(rng.standard_normal((5, 5)))
    po.write_rpcf(str(tmp_path / "a.rpcf"), f, [3, 1, 4, 1, 5], c)
    f2, p2, c2 = po.read_rpcf(str(tmp_path / "a.rpcf"))
    assert np.array_equal(f, f2) and list(p2) == [3, 1, 4, 1, 5] and np.array_equal(c, c2)
    assert os.path.getsize(tmp_path / "a.rpcf") == 24 + 8 * 37 * 5 + 8 * 5 + 8 + 8 * 15
    po.write_rpcf(str(tmp_path / "e.rpcf"), np.zeros((4, 0)), [], None)  # rank 0: no chol
    f3, p3, c3 = po.read_rpcf(str(tmp_path / "e.rpcf"))
    assert f3.shape == (4, 0) and p3.size == 0 and c3 is None
    with pytest.raises(ValueError):
        po.write_rpcf(str(tmp_path / "bad.rpcf"), f, [1, 2], c)


@pytest.fixture(scope="module")
def ctx():
    from paper_2410_03969_b200 import api
    c = api.Context(0)
    yield c
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k,b", [(20000, 10, 200, 40), (70000, 5, 300, 120), (3, 1, 3, 2)])
def test_gpu_rpcf_bytes(ctx, tmp_path, n, d, k, b):
    from paper_2410_03969_b200 import api
    x = wl.gen_c1(n, d, 0)
    g = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec("gaussian", math.sqrt(d))),
                                   api.RunConfig.until_rank(k, b, 0), ctx)
    g.write_rpcf(str(tmp_path / "gpu.rpcf"))
    g.write_trace_csv(str(tmp_path / "gpu.csv"))
    po.write_rpcf(str(tmp_path / "po.rpcf"), g.factor, g.pivots, g.chol_factor)
    po.write_pivot_trace_csv(str(tmp_path / "po.csv"), g.proposed, g.accepted)
    assert (tmp_path / "gpu.rpcf").read_bytes() == (tmp_path / "po.rpcf").read_bytes()
    assert (tmp_path / "gpu.csv").read_text() == (tmp_path / "po.csv").read_text()
    if pyref.available():
        f, p, c = pyref.read_rpcf(str(tmp_path / "gpu.rpcf"))
        assert np.array_equal(f, g.factor) and np.array_equal(p, g.pivots)
        assert np.array_equal(c, g.chol_factor)


@pytest.mark.gpu
def test_gpu_rpcf_matches_reference_run(ctx, tmp_path):
    """The GPU file and the reference's file for the same config: identical header, pivots
    and trace; factor and chol within the north_star 1e-10."""
    from paper_2410_03969_b200 import api
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_c1.npz"))
    w = wl.CONFIGS["C1"]
    g = api.accelerated_rpcholesky(api.KernelOracle(w.points(), api.KernelSpec(w.kernel, w.sigma)),
                                   api.RunConfig.until_rank(w.k, w.b, w.seed), ctx)
    g.write_rpcf(str(tmp_path / "gpu.rpcf"))
    f, p, c = po.read_rpcf(str(tmp_path / "gpu.rpcf"))
    assert np.array_equal(p, z["pivots"])
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(c, z["chol"]) <= 1e-10
    assert rel(f.sum(axis=0), z["col_sums"]) <= 1e-10
    assert rel(f[:: max(1, f.shape[0] // 64)], z["factor_rows_probe"]) <= 1e-10


@pytest.mark.gpu
def test_gpu_rpcf_shard_invariant_and_lowmem_refused(tmp_path):
    from paper_2410_03969_b200 import api
    x = wl.gen_c1(30000, 8, 1)
    ko = api.KernelOracle(x, api.KernelSpec("gaussian", 2.5))
    cfg = api.RunConfig.until_rank(250, 50, 3)
    api.accelerated_rpcholesky(ko, cfg, api.Context(0)).write_rpcf(str(tmp_path / "p1.rpcf"))
    api.accelerated_rpcholesky(ko, cfg, api.Context(0, virtual_shards=3)).write_rpcf(
        str(tmp_path / "p3.rpcf"))
    assert (tmp_path / "p1.rpcf").read_bytes() == (tmp_path / "p3.rpcf").read_bytes()
    lm = api.accelerated_rpcholesky_lowmem(ko, cfg, api.Context(0))
    with pytest.raises(ValueError, match="no factor"):
        lm.write_rpcf(str(tmp_path / "lm.rpcf"))
