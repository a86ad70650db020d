#!/bin/bash
O=gpurun_out/gs; mkdir -p $O
for g in 2 3 4 2 3 4; do
  SMP_K1_GEN_SETS=$g timeout 300 python bench.py --config cfg1 --no-cpu-baseline --no-e2e > $O/cfg1_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/cfg1_g$g.json'));r=d['roofline'];print('cfg1 gs=$g', round(d['sketch_ms'],4), round(r['k1_ms_per_launch'],4), d['clocks'])" >> $O/summary.log
done
for g in 3 4 2; do
  SMP_K1_GEN_SETS=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/cfg2_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/cfg2_g$g.json'));r=d['roofline'];print('cfg2 gs=$g', round(d['sketch_ms'],4), round(r['k1_ms_per_launch'],4), d['clocks'])" >> $O/summary.log
done
