#!/bin/bash
O=gpurun_out/t2; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "extreme" > $O/pytest_extreme.log 2>&1; tail -15 $O/pytest_extreme.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --config cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; tail -c 600 $O/bench_cfg4.json
