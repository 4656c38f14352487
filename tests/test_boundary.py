"""C-ABI boundary checks that need no GPU: the library builds, loads, and
exports every symbol include/rpchol_gpu.h declares; the host API mirrors the
reference's argument validation."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "rpchol_gpu.h")).read()
    return sorted(set(re.findall(r"\b(rpc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2410_03969_b200 import _lib
    lib = _lib.load()
    declared = header_symbols()
    assert declared, "no symbols parsed from the header"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess
    from paper_2410_03969_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass   # FP64 tensor-core path present


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_03969_b200 import api
    with pytest.raises(RuntimeError):
        api.Context(0)


def test_runconfig_validation():
    from paper_2410_03969_b200 import api
    with pytest.raises(ValueError):
        api.RunConfig.until_rank(0, 4, 0)
    with pytest.raises(ValueError):
        api.RunConfig.fixed_rounds(3, 0, 0)


def test_bench_gpus_flag_spawns_ranks_or_fails_loudly():
    """bench.py --gpus N (no torchrun) starts one process per GPU; with fewer GPUs visible it
    must fail with a message instead of silently running one rank."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("multi-GPU host: the spawn path would really run")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "--gpus 2" in r.stderr and "CUDA device" in r.stderr
