#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python scripts/bench_c5.py --layers 32 --batch 8 --prefix 2048 8192 32768 --k 16 64 --replays 3 > gpurun_out/c5_32l.jsonl 2> gpurun_out/c5.err
timeout 1500 python scripts/bench_c3.py > gpurun_out/c3.json 2> gpurun_out/c3.err
