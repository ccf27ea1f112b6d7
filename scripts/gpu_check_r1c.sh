#!/bin/bash
# Re-entry check: GPU tests, smoke, default bench, attention ncu capture (C5 shape) + raw CSV.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 8 -c 1 \
    -o gpurun_out/attn_tc_c5 python scripts/bench_c5.py --layers 4 --prefix 8192 --k 16 --replays 1 > gpurun_out/ncu_c5.log 2>&1
ncu -i gpurun_out/attn_tc_c5.ncu-rep --page raw --csv > gpurun_out/attn_tc_c5_raw.csv 2>/dev/null
ncu -i gpurun_out/attn_tc_c5.ncu-rep --page details --csv > gpurun_out/attn_tc_c5_details.csv 2>/dev/null
ls -la gpurun_out
