O=gpurun_out/probe9; mkdir -p $O
RPC_DEBUG_TRACE=1 python tools/one_factor.py C4 1 > $O/trace.txt 2>&1
echo done
