"""C++ drop-in: the reference's own KernelOracle/RunConfig/CholeskyResult types, its
CPU accelerated_rpcholesky (headers compiled against the Eigen-API shim) and
rpchol::b200::accelerated_rpcholesky (include/rpchol_b200.hpp over the C-ABI) on the
same inputs — pivots, PivotTrace, factor, chol_factor, residual diagonal and trace error
must agree (tests/cpp/dropin_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "DROPIN OK" in out.stdout


def test_dropin_binary_links_product_library():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built")
    ldd = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "librpchol_b200.so" in ldd and "not found" not in ldd.split("librpchol_b200.so")[1].split("\n")[0]
