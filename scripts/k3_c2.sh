#!/bin/bash
# K3 at the steady-state C2 batch shapes (rotations 68-77 of the bench workload): per-batch device
# time, and one ncu capture of a large and of a small batch
mkdir -p gpurun_out
timeout 600 python scripts/c2_attn_shapes.py gpurun_out/c2_shapes_ss.json 10 67 > gpurun_out/c2_shapes_ss.log 2>&1
timeout 600 python scripts/bench_attn.py --shapes gpurun_out/c2_shapes_ss.json --reps 20 > gpurun_out/k3_c2_ss.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 3 -c 1 -o gpurun_out/k3c2_b0 \
  python scripts/bench_attn.py --shapes gpurun_out/c2_shapes_ss.json --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/k3c2_b0.ncu-rep --page raw --csv > gpurun_out/k3c2_b0_raw.csv 2>/dev/null
cat gpurun_out/c2_shapes_ss.log; cat gpurun_out/k3_c2_ss.jsonl | cut -c1-250
