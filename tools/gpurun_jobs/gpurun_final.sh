#!/bin/bash
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --config cfg1 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --config cfg4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
