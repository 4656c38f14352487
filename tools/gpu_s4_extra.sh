#!/bin/bash
# Session-4 extras: int8 threshold sweep, the other configs' bench lines, scaling projection,
# ncu captures of the two-pass int8 GEMM and the update kernel (C4 round 9).
O=gpurun_out/${1:-s4_extra}; mkdir -p $O
for k in 192 256 384; do echo "MINK $k $(RPC_I8_MIN_K=$k timeout 200 python tools/i8_check.py C4 2>&1 | grep 'i8 fact')"; done > $O/mink.txt 2>&1
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-parity --no-cpu > $O/bench_C5.json 2> $O/bench_C5.err
for c in C2 C3 C1; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-parity --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python tools/scaling_projection.py > $O/scaling_projection.json 2> $O/scaling.err
bash tools/gpu_i8_profile.sh ${1:-s4_extra}
echo done
