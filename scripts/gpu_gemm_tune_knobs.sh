#!/bin/bash
# A/B of the algorithm-table search width (GLMX_GEMM_TUNE="candidates,rounds") on the C2 bench
mkdir -p gpurun_out
for i in 1 2 3; do
  python bench.py --no-cpu-baseline --no-standalone --decode-steps 0 > gpurun_out/kn_6_3_$i.json 2>/dev/null
  GLMX_GEMM_TUNE=12,5 python bench.py --no-cpu-baseline --no-standalone --decode-steps 0 > gpurun_out/kn_12_5_$i.json 2>/dev/null
done
for f in gpurun_out/kn_*.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['config']['gemm_algorithms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
