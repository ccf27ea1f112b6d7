#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/engine_tests.log 2>&1; echo "rc=$?" >> gpurun_out/engine_tests.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/decode64_launches.csv python scripts/decode_launches.py 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/decode64_launches.csv > gpurun_out/decode64_summary.txt 2>&1
