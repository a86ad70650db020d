#!/bin/bash
# Round-2 final K1 captures after the generator-set change (cfg2 default bench).
O=gpurun_out/prof2; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
  --kernel-name-base demangled --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "exit $?" >> $O/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_tc_kernel -s 2 -c 1 -o $O/k1_cfg2_r2c \
  python tools/prof_k1.py cfg2 1 > $O/ncu_k1_cfg2.log 2>&1
echo "exit $?" >> $O/ncu_k1_cfg2.log
