#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_append.py tests/test_gpu_engine.py -x -q > gpurun_out/append_tests.log 2>&1; echo "rc=$?" >> gpurun_out/append_tests.log
timeout 300 python scripts/bench_kernels.py --skip K2g K4 K1 > gpurun_out/kernels_k2.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
