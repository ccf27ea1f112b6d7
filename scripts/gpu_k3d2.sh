#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_engine.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/bench_attn.py --impl 2 --prefix 300 1500 3000 --suffix 1 --batch 8 64 128 > gpurun_out/decode_attn_impl2.jsonl 2>&1
for i in 1 2; do timeout 300 python scripts/decode_profile.py > gpurun_out/dp_$i.txt 2>&1; done
