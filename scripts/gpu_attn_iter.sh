#!/bin/bash
# Attention iteration: kernel parity tests, kernel sweep (tc vs mma), engine GPU tests, bench.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/bench_attn.py --check --prefix 2048 8192 32768 --suffix 128 --batch 8 > gpurun_out/attn_sweep_tc.jsonl 2>&1
timeout 300 python scripts/bench_attn.py --prefix 32768 --suffix 128 --batch 1 2 >> gpurun_out/attn_sweep_tc.jsonl 2>&1
timeout 300 python scripts/bench_attn.py --impl 1 --prefix 2048 8192 32768 --suffix 128 --batch 8 > gpurun_out/attn_sweep_mma.jsonl 2>&1
if [ "$1" == "full" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
