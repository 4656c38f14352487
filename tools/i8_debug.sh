#!/bin/bash
# Bound decomposition of i8gemm2_kernel at C4: full, without TMA loads, without products
# (RPC_I8_DEBUG; the factorization's results are wrong in modes 1-3, only the kernel times count).
O=gpurun_out/${1:-i8dbg}; mkdir -p $O
for d in ${2:-0 1 2 3 7 11 15}; do
  RPC_I8_DEBUG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:i8gemm2 -c 1 --csv \
    --log-file $O/dbg$d.csv python tools/one_c4.py > $O/dbg$d.log 2>&1
  echo "dbg $d: $(grep i8gemm2 $O/dbg$d.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
