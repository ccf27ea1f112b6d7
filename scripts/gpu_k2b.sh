#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_append.py tests/test_gpu_engine.py -x -q > gpurun_out/append_tests.log 2>&1; echo "rc=$?" >> gpurun_out/append_tests.log
timeout 300 python scripts/bench_kernels.py --skip K2g K4 K1 > gpurun_out/kernels_k2.jsonl 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/decode64_launches.csv python scripts/decode_launches.py 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/decode64_launches.csv > gpurun_out/decode64_summary.txt 2>&1
