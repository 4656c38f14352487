O=gpurun_out/probe11; mkdir -p $O
python tools/colbench.py C4 > $O/default.txt 2>&1
RPC_COLS_WC1=1 python tools/colbench.py C4 > $O/wc1.txt 2>&1
echo done
