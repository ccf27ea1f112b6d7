#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/bench_attn.py --shapes profiles/r1_c2_attn_shapes.json > gpurun_out/c2_attn_now.jsonl 2>&1
timeout 1200 python scripts/bench_c5.py --layers 32 --batch 8 --prefix 2048 8192 32768 --k 16 64 --replays 3 > gpurun_out/c5_32l.jsonl 2> gpurun_out/c5.err
