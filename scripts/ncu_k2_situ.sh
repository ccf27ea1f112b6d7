#!/bin/bash
# K2 in the C2 step: ncu launch metrics of late-rotation launches (cold cache, serialised)
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:rope_kv_append -s 250 -c 30 --csv --log-file gpurun_out/k2_situ_launches.csv \
  python bench.py --no-cpu-baseline --steps 6 --warmup 3 --decode-steps 0 > gpurun_out/k2_situ.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 6 --warmup 3 --decode-steps 0 > gpurun_out/k2_situ_bench.json 2>&1
