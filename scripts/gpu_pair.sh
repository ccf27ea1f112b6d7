#!/bin/bash
# K3 paired single-tile items: parity tests, C2 / decode shapes with pairing on and off, bench.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
for P in 1 0; do
  GLMX_ATTN_PAIR=$P timeout 300 python scripts/bench_attn.py --shapes profiles/r1_c2_attn_shapes.json > gpurun_out/c2_attn_pair$P.jsonl 2>&1
  GLMX_ATTN_PAIR=$P timeout 300 python scripts/bench_attn.py --prefix 300 2000 --suffix 1 8 --batch 64 200 > gpurun_out/decode_attn_pair$P.jsonl 2>&1
done
if [ "$1" == "full" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
  for P in 1 0; do
    GLMX_ATTN_PAIR=$P timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pair$P.json 2> gpurun_out/bench_pair$P.err
  done
  GLMX_ATTN_PAIR=1 timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile_pair1.txt 2>&1
  GLMX_ATTN_PAIR=0 timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile_pair0.txt 2>&1
fi
