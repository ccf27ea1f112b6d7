#!/bin/bash
# K3 at the low-prefix C5 cells: kernel-level bench + an ncu launch list of the same shapes
mkdir -p gpurun_out
timeout 600 python scripts/bench_attn.py --prefix 2048 4096 8192 --suffix 80 104 --batch 8 --reps 20 > gpurun_out/k3_lowp.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/k3_lowp_launches.csv python scripts/bench_attn.py --prefix 2048 --suffix 104 --batch 8 --reps 2 > /dev/null 2>&1
cat gpurun_out/k3_lowp.jsonl
