#!/bin/bash
# compute-sanitizer memcheck over the kernel-level parity tests (small shapes)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --target-processes all \
  python -m pytest tests/test_gpu_chunks.py tests/test_gpu_append.py -x -q > gpurun_out/memcheck_k1k2.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_k1k2.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_attention.py -x -q -k "decode or paired or mixed" > gpurun_out/memcheck_k3.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_k3.log
