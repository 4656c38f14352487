O=gpurun_out/r7; mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
for c in C1 C2 C3 C4 C5; do python tools/one_factor.py $c 3 2>&1 | tail -1 >> $O/configs.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:update_kernel -s 9 -c 1 \
  -o $O/upd_r9 python tools/one_factor.py C4 1 > $O/ncu_full.log 2>&1
echo done
