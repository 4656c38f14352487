#!/bin/bash
# Bound decomposition of i8gemm2_kernel at C4: the first tensor-core launch timed
# by ncu under RPC_I8_DEBUG bit masks (1 no TMA loads, 2 no products, 4 no C stores, 8 no
# conversions; results are wrong in those modes, only the kernel times count).  Set
# RPC_I8_MIN_K=900 to make that first launch the nkb = 15 one.
#   gpurun -- 'RPC_I8_MIN_K=900 bash tools/i8_debug.sh i8dbg "0 1 2 3"' 
O=gpurun_out/${1:-i8dbg}; mkdir -p $O
for d in ${2:-0 1 2 3 7 11 15}; do
  RPC_I8_DEBUG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:i8gemm2 -c 1 --csv \
    --log-file $O/dbg$d.csv python tools/one_c4.py > $O/dbg$d.log 2>&1
  echo "dbg $d: $(grep i8gemm2 $O/dbg$d.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
