#!/bin/bash
# K2 check: append/engine GPU tests, the K2 kernel bench and a C2 bench line (in-step K2 fraction).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_append.py tests/test_gpu_engine.py -q -x > gpurun_out/pytest_k2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k2.log
timeout 300 python scripts/bench_kernels.py --skip K1 K2g K4 > gpurun_out/k2_kernels.jsonl 2> gpurun_out/k2_kernels.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_k2.json 2> gpurun_out/bench_k2.err
tail -3 gpurun_out/pytest_k2.log; cat gpurun_out/k2_kernels.jsonl | head -5
