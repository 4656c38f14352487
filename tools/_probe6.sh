O=gpurun_out/probe6; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden_fixtures.py -m gpu -x -q > $O/pytest.txt 2>&1
RPC_DEBUG_TRACE=1 python tools/one_factor.py C4 1 > $O/trace.txt 2>&1
python tools/one_factor.py C4 3 > $O/c4.txt 2>&1
python tools/one_factor.py C2 3 >> $O/c4.txt 2>&1
python tools/one_factor.py C3 3 >> $O/c4.txt 2>&1
echo done
