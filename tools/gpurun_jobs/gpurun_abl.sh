#!/bin/bash
O=gpurun_out/f32; mkdir -p $O
for v in $VARS; do
SMP_LIB=/root/repo/paper_1610_06656_b200/libsmp_$v.so timeout 300 python tools/k1f_ablation.py 10 $MODES 2>&1 | grep mode | tee -a $O/k1f_ablation4.log
done
