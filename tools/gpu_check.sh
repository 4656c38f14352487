#!/bin/bash
# One gpurun pass over the current tree: GPU tests, smoke, bench (both arms), launch list.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-check}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
# (ncu only right after the identical command exited 0 without it)
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $O/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu.log 2>&1
echo done
