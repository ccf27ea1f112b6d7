#!/bin/bash
# C2 attention shapes: dump them, time K3 (tc, mma) on them, ncu one mid-run batch.
mkdir -p gpurun_out
timeout 600 python scripts/c2_attn_shapes.py gpurun_out/c2_shapes.json 11 > gpurun_out/c2_shapes.log 2>&1
timeout 300 python scripts/bench_attn.py --shapes gpurun_out/c2_shapes.json > gpurun_out/c2_attn_tc.jsonl 2>&1
timeout 300 python scripts/bench_attn.py --impl 1 --shapes gpurun_out/c2_shapes.json > gpurun_out/c2_attn_mma.jsonl 2>&1
python - <<'PY'
import json
b = json.load(open("gpurun_out/c2_shapes.json"))
json.dump([b[6]], open("gpurun_out/c2_one.json", "w"))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 3 -c 1 \
    -o gpurun_out/attn_c2 python scripts/bench_attn.py --shapes gpurun_out/c2_one.json --reps 1 > gpurun_out/attn_c2_ncu.log 2>&1
ncu -i gpurun_out/attn_c2.ncu-rep --page raw --csv > gpurun_out/attn_c2_raw.csv 2>/dev/null
ncu -i gpurun_out/attn_c2.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_c2_sass.csv 2>/dev/null
