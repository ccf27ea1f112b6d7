#!/bin/bash
# Round-1 profiling: launch list of one timed bench rotation + full ncu capture of the hot kernels.
mkdir -p gpurun_out
# ~200 init launches + ~420 per rotation: skip init + 2 warm-up rotations, list one rotation.
ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 500 --csv \
    --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 100 -c 2 \
    -o gpurun_out/attn_tc_r1 python bench.py --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/attn_run.log 2>&1
ls -la gpurun_out
