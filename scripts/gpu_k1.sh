#!/bin/bash
# K1 iteration: chunk parity tests, K1 sweep, launch list of the K1 sweep.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chunks.py tests/test_retrieve_node.py -x -q > gpurun_out/chunk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chunk_tests.log
timeout 300 python scripts/bench_kernels.py --skip K2 K2g K4 > gpurun_out/kernels_k1.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/k1_launches.csv python scripts/bench_kernels.py --skip K2 K2g K4 --reps 4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/k1_launches.csv > gpurun_out/k1_launch_summary.txt 2>&1
