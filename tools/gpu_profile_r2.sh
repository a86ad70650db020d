#!/bin/bash
# One gpurun job: sanitizers on small shapes, the default bench, the ncu launch
# list of the default bench, and ncu --set full captures of the dominant
# kernels (K1 at cfg1/cfg2, K3 stages at cfg3).  Outputs in gpurun_out/r2/.
O=gpurun_out/r2
mkdir -p $O
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $O/sanitize_$tool.log 2>&1
  echo "exit $?" >> $O/sanitize_$tool.log
done
python bench.py > $O/bench_default.json 2> $O/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sketch_tc_kernel -s 2 -c 1 -o $O/k1_cfg2_r2 \
    python tools/prof_k1.py cfg2 1 > $O/ncu_k1_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sketch_tc_kernel -s 4 -c 1 -o $O/k1_cfg1_r2 \
    python tools/prof_k1.py cfg1 2 > $O/ncu_k1_cfg1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:csr_|pi_panel|pi_transpose|sketch_tc" -s 40 -c 9 -o $O/k3_cfg3_r2 \
    python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_k3.log 2>&1
