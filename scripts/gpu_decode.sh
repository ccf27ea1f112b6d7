#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_engine.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
for I in 2 0; do
  timeout 300 python scripts/bench_attn.py --impl $I --prefix 300 2000 --suffix 1 --batch 8 64 200 > gpurun_out/decode_attn_impl$I.jsonl 2>&1
done
timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile.txt 2>&1
GLMX_DECODE_ATTN=tc timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile_tc.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
