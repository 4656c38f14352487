#!/bin/bash
# Timing sweep of the two-pass int8 residual GEMM on C4: K-chunk sizes, CTA pair on / off.
for kc in 16 8 5 4; do
  echo "KCHUNK $kc pair"; RPC_I8_KCHUNK=$kc timeout 200 python tools/i8_check.py C4 2>&1 | grep "i8 fact\|dF\|pivots"
  echo "KCHUNK $kc onecta"; RPC_I8_ONECTA=1 RPC_I8_KCHUNK=$kc timeout 200 python tools/i8_check.py C4 2>&1 | grep "i8 fact"
done
