#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/g1.py <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import torch
from paper_2511_01633_b200.ops import gemv
for n in (8, 64):
    x = torch.randn((n, 4096), device="cuda").to(torch.bfloat16)
    w = torch.randn((6144, 4096), device="cuda").to(torch.bfloat16)
    y = torch.empty((n, 6144), device="cuda", dtype=torch.bfloat16)
    gemv(x, w, y, 0, reps=2)
PY
timeout 600 ncu --set full --clock-control none -k regex:gemv_tc -c 4 -o gpurun_out/gemv python /tmp/g1.py > gpurun_out/gemv_ncu.log 2>&1
ncu -i gpurun_out/gemv.ncu-rep --page raw --csv > gpurun_out/gemv_raw.csv 2>/dev/null
