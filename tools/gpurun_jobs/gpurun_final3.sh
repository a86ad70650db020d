#!/bin/bash
O=gpurun_out/final3; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python bench.py --config cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -c 3000 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
