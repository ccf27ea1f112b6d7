#!/bin/bash
# Round-1 profiling: launch list of one bench step + full ncu capture of the attention kernel.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1200 --csv \
    --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:paged_attn -s 40 -c 2 \
    -o gpurun_out/attn_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/attn_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"chunk_select|chunk_render|rope_kv|rmsnorm|swiglu" -s 10 -c 6 \
    -o gpurun_out/misc_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/misc_run.log 2>&1
ls -la gpurun_out
