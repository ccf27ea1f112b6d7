#!/bin/bash
# Final-round evidence runs on one B200: the 20-cell C5 grid in the engine, compute-sanitizer
# memcheck over the K3 / engine / chunk tests, racecheck over K1.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 2400 python scripts/bench_c5.py > gpurun_out/c5_grid_final.jsonl 2> gpurun_out/c5_grid_final.err
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py tests/test_gpu_append.py -x -q > gpurun_out/memcheck_k2k3.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_k2k3.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_engine.py tests/test_gpu_chunks.py -x -q > gpurun_out/memcheck_engine_k1.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_engine_k1.log
for f in memcheck_k2k3 memcheck_engine_k1; do echo "## $f"; grep -a -E "passed|SUMMARY|rc=" gpurun_out/$f.log; done
wc -l gpurun_out/c5_grid_final.jsonl
