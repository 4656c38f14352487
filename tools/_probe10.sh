O=gpurun_out/probe10; mkdir -p $O
RPC_DEBUG_TIMING=1 python tools/one_factor.py C4 2 > $O/wc2.txt 2>&1
RPC_NO_WC2=1 RPC_DEBUG_TIMING=1 python tools/one_factor.py C4 2 > $O/wc1.txt 2>&1
python tools/one_factor.py C2 2 > $O/c2wc2.txt 2>&1
RPC_NO_WC2=1 python tools/one_factor.py C2 2 > $O/c2wc1.txt 2>&1
echo done
