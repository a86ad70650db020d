#!/bin/bash
O=gpurun_out/t8; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "gauss or f32 or cfg4 or fp32 or pi_bit_exact or csr or extreme or lela" > $O/pytest_gauss.log 2>&1; tail -3 $O/pytest_gauss.log
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 8 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
python - <<PY
import json
l=[x for x in open("$O/bench_cfg4.json") if x.startswith("{")]
j=json.loads(l[-1]); print("cfg4", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["clocks"])
PY
