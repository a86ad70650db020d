#!/bin/bash
# K3 (cfg3) ncu captures: one panel's worth of kernels in full, the whole
# step's per-launch times and DRAM bytes; K1F at cfg4.  Outputs gpurun_out/r2p/.
O=gpurun_out/r2p
mkdir -p $O
ncu --set full --clock-control none -k "regex:csr_hist|csr_colscan|csr_scatter|csr_total|pi_panel_dual|csr_accumulate|DeviceScan" -s 40 -c 8 -o $O/k3_panel \
    python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_k3_panel.log 2>&1
ncu --set full --clock-control none -k "regex:csr_densify|sketch_tc_kernel|reduce_sketch" -s 3 -c 3 -o $O/k3_head \
    python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_k3_head.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/k3_step_metrics.csv python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
    > $O/ncu_k3_step.log 2>&1
ncu --set full --clock-control none -k regex:sketch_tc_f32 -s 1 -c 1 -o $O/k1f_cfg4 \
    python tools/prof_k1.py cfg4 1 > $O/ncu_k1f.log 2>&1
