#!/bin/bash
# HBM-bound kernels: parity (K2) + bandwidth sweep + launch list of the sweep (per-kernel times).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_append.py -x -q > gpurun_out/append_tests.log 2>&1; echo "rc=$?" >> gpurun_out/append_tests.log
timeout 600 python scripts/bench_kernels.py > gpurun_out/kernels.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/kernels_launches.csv python scripts/bench_kernels.py --reps 4 > gpurun_out/kernels_ncu.log 2>&1
