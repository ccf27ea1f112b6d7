#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k decode > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/bench_attn.py --impl 2 --prefix 300 1500 3000 --suffix 1 --batch 8 64 128 > gpurun_out/decode_attn_impl2.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-standalone > gpurun_out/bench.json 2> gpurun_out/bench.err
