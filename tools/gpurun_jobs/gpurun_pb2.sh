#!/bin/bash
O=gpurun_out/pb; mkdir -p $O
for b in 16 15 16; do
  SMP_CSR_PANEL_BITS=$b timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/cfg3_b$b.json 2> $O/cfg3_b$b.err
  python -c "import json;d=json.load(open('$O/cfg3_b$b.json'));r=d['roofline'];print('bits=$b', round(d['sketch_ms'],3), round(r['k3d_ms_per_launch'],4), round(r['l2_pi_gather_tb_s'],2), d['clocks'])" >> $O/summary2.log 2>&1
done
SMP_CSR_PANEL_BITS=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "csr" > $O/pytest_csr16.log 2>&1
echo "exit $?" >> $O/pytest_csr16.log
