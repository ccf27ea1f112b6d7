#!/bin/bash
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_engine.py -x -q -k "not c3_shaped" > gpurun_out/memcheck_engine.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_engine.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_chunks.py -x -q > gpurun_out/racecheck_k1.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_k1.log
