#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/bench_attn.py --shapes profiles/r1_c2_attn_shapes.json > gpurun_out/c2_attn_now.jsonl 2>&1
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
