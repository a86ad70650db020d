#!/bin/bash
O=gpurun_out/p1; mkdir -p $O
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sketch_tc_f32 -s 2 -c 1 -f -o $O/k1f_cfg4_r2c python tools/k1f_ablation.py 1 0 > $O/ncu_k1f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -c 3000 --csv --log-file $O/launches_cfg4.csv python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
ls -la $O
