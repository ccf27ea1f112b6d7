#!/bin/bash
# K3 at the short-prefix C5 cells: kernel sweep, launch list (attention + split combine) and one
# full capture at prefix 2048, suffix 104 (the k=16 cell's mean suffix).
mkdir -p gpurun_out
TAG=${TAG:-k3s}
timeout 300 python scripts/bench_attn.py --prefix 2048 4096 8192 --suffix 80 104 128 --reps 20 > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python scripts/bench_attn.py --prefix 2048 --suffix 104 --reps 2 > /dev/null 2>&1
P=2048 bash -c "timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 3 -c 1 -o gpurun_out/${TAG}_p2048 python scripts/bench_attn.py --prefix 2048 --suffix 104 --reps 1 > gpurun_out/${TAG}_ncu.log 2>&1"
ncu -i gpurun_out/${TAG}_p2048.ncu-rep --page raw --csv > gpurun_out/${TAG}_p2048_raw.csv 2>/dev/null
cat gpurun_out/${TAG}_sweep.jsonl
