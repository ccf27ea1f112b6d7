#!/bin/bash
# ncu --set full of K4 (local page copy) and K3d (decode attention) for profiles/
mkdir -p gpurun_out
cat > /tmp/k4.py <<'PY'
import sys, os, random, ctypes as C
sys.path.insert(0, os.getcwd())
import torch
import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200._lib import check, lib
n = 1024
kv = glmx.KvCacheState(2 * n + 16, 16, glmx.PRIORITY, device=0, n_layers=32, n_kv_heads=8, head_dim=128, headroom_pages=16)
src = list(range(n)); dst = list(range(n, 2 * n)); random.Random(1).shuffle(dst)
s_arr = (C.c_int32 * n)(*src); d_arr = (C.c_int32 * n)(*dst)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    check(lib().glmx_pool_copy(kv.h, kv.h, s_arr, d_arr, n, st))
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:pool_copy -s 2 -c 1 -o gpurun_out/k4 python /tmp/k4.py > gpurun_out/k4_ncu.log 2>&1
ncu -i gpurun_out/k4.ncu-rep --page raw --csv > gpurun_out/k4_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:decode_attn -s 2 -c 1 -o gpurun_out/k3d \
  python scripts/bench_attn.py --impl 2 --prefix 300 --suffix 1 --batch 64 --reps 1 > gpurun_out/k3d_ncu.log 2>&1
ncu -i gpurun_out/k3d.ncu-rep --page raw --csv > gpurun_out/k3d_raw.csv 2>/dev/null
