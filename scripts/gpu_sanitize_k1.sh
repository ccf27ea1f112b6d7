#!/bin/bash
# compute-sanitizer over the K1 parity tests (memcheck: out-of-bounds / misaligned; racecheck:
# shared-memory hazards of the staged text buffer) and the engine tests.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_chunks.py tests/test_retrieve_node.py -x -q > gpurun_out/memcheck_k1.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_k1.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_chunks.py -x -q -k "fixture or attribute or irregular" > gpurun_out/racecheck_k1.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_k1.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_engine.py -x -q -k "reuse or prefill_batch or decode_matches" > gpurun_out/memcheck_engine.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_engine.log
for f in memcheck_k1 racecheck_k1 memcheck_engine; do echo "## $f"; tail -4 gpurun_out/$f.log; done
