#!/bin/bash
O=gpurun_out/t3; mkdir -p $O
export SMP_LIB=/root/repo/paper_1610_06656_b200/libsmp_fd.so
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "f32" > $O/pytest_f32.log 2>&1; tail -3 $O/pytest_f32.log
timeout 200 python tools/k1f_ablation.py 10 0,69,0 2>&1 | grep mode | tee $O/abl.log
unset SMP_LIB
timeout 200 python tools/k1f_ablation.py 10 0 2>&1 | grep mode | tee -a $O/abl.log
