#!/bin/bash
# Reuse on/off A/B (bench.py --no-reuse) and the retrieval/prefill pipeline-law timing check.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x -k reuse_off > gpurun_out/pytest_reuse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_reuse.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/ab_reuse_on.json 2> gpurun_out/ab_reuse_on.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-standalone --no-reuse > gpurun_out/ab_reuse_off.json 2> gpurun_out/ab_reuse_off.err
timeout 900 python scripts/pipeline_law.py > gpurun_out/pipeline_law.json 2> gpurun_out/pipeline_law.err
tail -3 gpurun_out/pytest_reuse.log; tail -c 400 gpurun_out/ab_reuse_off.json; tail -c 600 gpurun_out/pipeline_law.err
