#!/bin/bash
O=gpurun_out/gs2; mkdir -p $O
for c in cfg1 cfg2; do for g in 2 3 4; do
SMP_K1_GEN_SETS=$g timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > $O/b_${c}_$g.json 2>/dev/null
python - <<PY
import json
l=[x for x in open("$O/b_${c}_$g.json") if x.startswith("{")]
j=json.loads(l[-1]); print("$c sets $g", round(j["sketch_ms"],3), round(j["roofline"]["k1_ms_per_launch"],4), j["clocks"]["sm_mhz"], j["clocks"]["reasons"])
PY
done; done | tee $O/gen_sets_final.log
