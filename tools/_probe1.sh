O=gpurun_out/probe1; mkdir -p $O
./tools/dmma_mix > $O/dmma_mix.txt 2>&1
RPC_DEBUG_TIMING=1 python tools/one_factor.py C4 3 > $O/timing.txt 2>&1
RPC_DEBUG_PHASES=1 python tools/one_factor.py C4 1 > $O/phases.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:update_kernel -s 10 -c 1 \
  -o $O/upd_r10 python tools/one_factor.py C4 1 > $O/ncu_full.log 2>&1
echo done
