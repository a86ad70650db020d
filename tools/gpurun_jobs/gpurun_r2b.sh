#!/bin/bash
O=gpurun_out/r2b
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "generator_sets" > $O/pytest_gensets.log 2>&1
echo "exit $?" >> $O/pytest_gensets.log
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --config cfg1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "exit $?" >> $O/pytest_gpu.log
