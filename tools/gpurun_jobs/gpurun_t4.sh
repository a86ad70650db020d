#!/bin/bash
O=gpurun_out/t4; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "pi_bit_exact or sketch_bf16 or generator_sets or srht or unaligned or hadamard or a_equals_b or csr or shard or zero" > $O/pytest_k1.log 2>&1; tail -3 $O/pytest_k1.log
for c in cfg1 cfg2; do
timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
python - <<PY
import json
l=[x for x in open("$O/bench_$c.json") if x.startswith("{")]
j=json.loads(l[-1]); print("$c", j["sketch_ms"], j["roofline"]["k1_ms_per_launch"], j["roofline"]["frac"], j["roofline_pct_of_stage"], j["clocks"])
PY
done
