#!/bin/bash
# K1 generator-set / mbarrier-wait variants (tuning experiment)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/k1v.log
for v in libsmp libsmp_g4 libsmp_ns libsmp_g3 libsmp_g4ns; do
  SMP_LIB=paper_1610_06656_b200/$v.so timeout 300 python tools/k1_ablation.py cfg2 12 0,5,1 >> gpurun_out/k1v.log 2>&1
  SMP_LIB=paper_1610_06656_b200/$v.so timeout 200 python tools/k1_ablation.py cfg1 300 0,5,1 >> gpurun_out/k1v.log 2>&1
done
SMP_LIB=paper_1610_06656_b200/libsmp_g4.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sketch_bf16 or pi_bit_exact or srht_parity or unaligned or a_equals_b" > gpurun_out/k1v_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/k1v_pytest.log
