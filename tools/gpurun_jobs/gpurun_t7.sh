#!/bin/bash
O=gpurun_out/t7; mkdir -p $O
for pb in 1 2 16; do
SMP_F32_PANEL_BLOCKS=$pb timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 8 > $O/bench_cfg4_pb$pb.json 2> $O/bench_cfg4_pb$pb.err
python - <<PY
import json
l=[x for x in open("$O/bench_cfg4_pb$pb.json") if x.startswith("{")]
j=json.loads(l[-1]); print("panel blocks/SM $pb", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["clocks"])
PY
done
SMP_F32_PANEL_OVERLAP=0 timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 8 2>/dev/null | python -c "
import sys,json
l=[x for x in sys.stdin if x.startswith('{')]; j=json.loads(l[-1]); print('serial', j['sketch_ms'], j['roofline']['k1_ms_per_launch'])"
timeout 900 python -m pytest tests -m gpu -x -q -k "f32 or cfg4 or fp32 or cfg0 or tiny or extreme or lela or a_equals_b" > $O/pytest_f32.log 2>&1; tail -3 $O/pytest_f32.log
