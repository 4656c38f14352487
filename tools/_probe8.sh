O=gpurun_out/probe8; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden_fixtures.py -m gpu -x -q > $O/pytest.txt 2>&1
for c in C2 C3 C4; do python tools/one_factor.py $c 3 2>&1 | tail -1 >> $O/t.txt; done
echo done
