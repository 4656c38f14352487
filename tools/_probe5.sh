O=gpurun_out/probe5; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
RPC_DEBUG_TIMING=1 python tools/one_factor.py C4 3 > $O/timing.txt 2>&1
python tools/one_factor.py C2 3 >> $O/timing.txt 2>&1
python tools/one_factor.py C3 3 >> $O/timing.txt 2>&1
python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err
echo done
python bench.py --variant lowmem --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/probe5/lowmem.json 2> gpurun_out/probe5/lowmem.err
python tools/matvec_probe.py > gpurun_out/probe5/matvec.txt 2>&1
