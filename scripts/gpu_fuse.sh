#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile.txt 2>&1
GLMX_DECODE_ATTN=unfused timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile_unfused.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-standalone > gpurun_out/bench.json 2> gpurun_out/bench.err
