#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/l2_probe.py --save > gpurun_out/l2_probe.log 2>&1
echo "exit $?" >> gpurun_out/l2_probe.log
