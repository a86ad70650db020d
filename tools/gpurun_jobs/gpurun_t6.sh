#!/bin/bash
O=gpurun_out/t6; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "f32 or cfg4 or fp32 or cfg0 or tiny or extreme or lela or a_equals_b" > $O/pytest_f32.log 2>&1; tail -3 $O/pytest_f32.log
for ov in 1 0; do
SMP_F32_PANEL_OVERLAP=$ov timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 8 > $O/bench_cfg4_ov$ov.json 2> $O/bench_cfg4_ov$ov.err
python - <<PY
import json
l=[x for x in open("$O/bench_cfg4_ov$ov.json") if x.startswith("{")]
j=json.loads(l[-1]); print("overlap $ov", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["clocks"])
PY
done
