#!/bin/bash
# ncu --set full captures of K1 (emit, 65k chunks), K2 gather (16k pages), K5 (100k-row scan) and a
# 32-layer C5 forward sweep.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:chunk_emit -s 8 -c 1 -o gpurun_out/k1_emit_v2 python scripts/bench_kernels.py --reps 4 --skip K2 K4 K2g > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:kv_gather_tma -s 4 -c 1 -o gpurun_out/k2_gather python scripts/bench_kernels.py --reps 1 --skip K1 K2 K4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:nearest_kernel -s 2 -c 1 -o gpurun_out/k5_nearest python scripts/workload_scale.py 100000 > /dev/null 2>&1
for f in k1_emit_v2 k2_gather k5_nearest; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
timeout 1500 python scripts/bench_c5.py --layers 32 --prefix 8192 32768 --k 16 > gpurun_out/c5_32l.jsonl 2>&1
