#!/bin/bash
# Full ncu capture of one K3 launch at a C5 shape (prefix $1, suffix $3 [128], batch $4 [8]) +
# raw/source CSV.
P=${1:-8192}; TAG=${2:-attn_tc}; S=${3:-128}; B=${4:-8}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 3 -c 1 \
    -o gpurun_out/${TAG}_p${P} python scripts/bench_attn.py --prefix $P --suffix $S --batch $B --reps 1 > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_p${P}.ncu-rep --page raw --csv > gpurun_out/${TAG}_p${P}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_p${P}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_p${P}_sass.csv 2>/dev/null
