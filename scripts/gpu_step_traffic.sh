#!/bin/bash
# Launch list of bench.py's timed C2 step with DRAM bytes per launch (ncu, profiler range = the
# timed rotations; cold-cache serialised per-launch times) -> the per-class traffic bench.py
# reports (profiles/r2_c2_traffic.json) and the launch summary.
mkdir -p gpurun_out
GLMX_PROFILE_RANGE=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/r2_c2_step_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/r2_c2_step_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/r2_c2_step_launches.csv --traffic gpurun_out/r2_c2_traffic.json > gpurun_out/r2_c2_step_summary.txt 2>&1
tail -5 gpurun_out/r2_c2_step_summary.txt; cat gpurun_out/r2_c2_traffic.json
