#!/bin/bash
O=gpurun_out/comb; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_abi.py -m "gpu or not gpu" -x -q > $O/pytest_shards.log 2>&1
echo "exit $?" >> $O/pytest_shards.log
