#!/bin/bash
# K1 barrier back-off sweep (tuning experiment)
O=gpurun_out/bo; mkdir -p $O
for b in 0 64 256 1000; do
  SMP_K1_BACKOFF_NS=$b timeout 300 python tools/k1_ablation.py cfg2 12 0,5,0 2>&1 | grep -v Warn | sed "s/^/bo=$b /" >> $O/k1_backoff.log
  SMP_K1_BACKOFF_NS=$b timeout 200 python tools/k1_ablation.py cfg1 300 0,5,0 2>&1 | grep -v Warn | sed "s/^/bo=$b /" >> $O/k1_backoff.log
done
SMP_K1_BACKOFF_NS=256 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sketch_bf16 or generator_sets or unaligned or a_equals_b or srht" > $O/pytest_bo.log 2>&1
echo "exit $?" >> $O/pytest_bo.log
