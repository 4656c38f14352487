#!/bin/bash
# ncu captures of the C4 round-9 launches in the tensor-core residual build: the fused update
# kernel (FP64 part) and the int8 residual GEMM (each only after the plain run succeeded).
O=gpurun_out/${1:-i8prof}
mkdir -p $O
timeout 300 python tools/one_c4.py > $O/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:i8gemm -s 4 -c 1 \
  -o $O/i8gemm_r9 python tools/one_c4.py > $O/ncu_i8.log 2>&1
if [ -n "$2" ]; then
RPC_I8_ONECTA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:i8gemm -s 4 -c 1 \
  -o $O/i8gemm_r9_onecta python tools/one_c4.py > $O/ncu_i8_1.log 2>&1
fi
if [ -z "$2" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:update_kernel -s 9 -c 1 \
  -o $O/update_r9_tc python tools/one_c4.py > $O/ncu_update.log 2>&1
fi
echo done
