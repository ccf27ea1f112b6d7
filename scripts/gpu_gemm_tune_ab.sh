#!/bin/bash
# A/B of the cuBLAS algorithm table (glmx_model_tune_gemms) on the C2 bench: alternating runs
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -q -m gpu -k "tuned or llama8b" 2>&1 | tail -3
for i in 1 2; do
  python bench.py --no-cpu-baseline --no-standalone > gpurun_out/ab_tuned_$i.json 2> gpurun_out/ab_tuned_$i.err
  python bench.py --no-cpu-baseline --no-standalone --gemm-tune-tokens 0 > gpurun_out/ab_default_$i.json 2> gpurun_out/ab_default_$i.err
done
for f in gpurun_out/ab_*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['graph_cot_queries_per_s']['value'] if d.get('graph_cot_queries_per_s') else None, d['config']['gemm_algorithms'], d['clocks'])"
done
