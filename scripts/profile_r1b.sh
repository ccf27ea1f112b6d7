#!/bin/bash
# Full ncu capture of the tcgen05 attention kernel (one launch of a C5-shaped batch) + C5 sweep.
mkdir -p gpurun_out
timeout 600 python scripts/bench_c5.py --layers 4 --prefix 2048 8192 32768 --k 16 64 > gpurun_out/c5_tc.jsonl 2>&1
GLMX_ATTN=mma timeout 600 python scripts/bench_c5.py --layers 4 --prefix 2048 8192 32768 --k 16 64 > gpurun_out/c5_mma.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn -s 8 -c 1 \
    -o gpurun_out/attn_tc_c5 python scripts/bench_c5.py --layers 4 --prefix 8192 --k 16 --replays 1 > gpurun_out/ncu_c5.log 2>&1
ls -la gpurun_out
