#!/bin/bash
O=gpurun_out/f32; mkdir -p $O
for m in 197 0; do
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sketch_tc_f32 -s 2 -c 1 -f -o $O/k1f_m$m python tools/k1f_ablation.py 1 $m > $O/ncu_m$m.log 2>&1
done
ls -la $O
