#!/bin/bash
O=gpurun_out/t1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "f32 or cfg4 or fp32 or gauss or cfg0 or shard or lela or table1 or tiny" > $O/pytest_f32.log 2>&1; tail -3 $O/pytest_f32.log
timeout 300 python tools/k1f_ablation.py 10 0,1,0 2>&1 | grep mode | tee $O/abl.log
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; python - <<PY
import json
l=[x for x in open("$O/bench_cfg4.json") if x.startswith("{")]
j=json.loads(l[-1]); print("cfg4", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["clocks"])
PY
