#!/bin/bash
O=gpurun_out/f32
mkdir -p $O
for v in $EXTRA; do
  L=/root/repo/paper_1610_06656_b200/libsmp$v.so
  SMP_LIB=$L timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e --steps 5 > $O/bench_cfg4$v.json 2> $O/bench_cfg4$v.err
  python - <<PY
import json
l=[x for x in open("$O/bench_cfg4$v.json") if x.startswith("{")]
j=json.loads(l[-1]); print("variant '$v'", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["clocks"])
PY
done
for v in $EXTRA; do
  SMP_LIB=/root/repo/paper_1610_06656_b200/libsmp$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "f32 or cfg4 or fp32 or gauss" 2>&1 | tail -2
done
