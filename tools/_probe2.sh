O=gpurun_out/probe2; mkdir -p $O
for s in 0 25 50 75 0 50; do echo "stagger $s" >> $O/stagger.txt; RPC_STAGGER=$s python tools/one_factor.py C4 4 2>&1 | tail -3 >> $O/stagger.txt; done
for s in 0 50; do echo "C2 stagger $s" >> $O/stagger.txt; RPC_STAGGER=$s python tools/one_factor.py C2 4 2>&1 | tail -2 >> $O/stagger.txt; done
echo done
