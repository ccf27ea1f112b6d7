#!/bin/bash
# GPU parity suite + smoke + a short C2 bench (one box): logs under gpurun_out/.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
if [ -n "$WITH_BENCH" ]; then
  timeout 900 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
fi
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
