#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemv.py -x -q > gpurun_out/gemv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gemv_tests.log
timeout 300 python - > gpurun_out/gemv_bench.txt 2>&1 <<'PY'
import torch, json
from paper_2511_01633_b200.ops import gemv
for K, N in [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096), (4096, 128256)]:
    for n in (8, 64):
        x = torch.randn((n, K), device="cuda").to(torch.bfloat16)
        w = torch.randn((N, K), device="cuda").to(torch.bfloat16)
        y = torch.empty((n, N), device="cuda", dtype=torch.bfloat16)
        gemv(x, w, y, 0, reps=3)
        ms = gemv(x, w, y, 0, reps=20)
        # cuBLAS reference time (torch.matmul -> cublas)
        for _ in range(3): torch.matmul(x, w.T)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): torch.matmul(x, w.T)
        e1.record(); torch.cuda.synchronize()
        cb = e0.elapsed_time(e1) / 20
        by = N * K * 2
        print(json.dumps({"K": K, "N": N, "n": n, "ms": ms, "gbs": by / ms / 1e6, "cublas_ms": cb, "cublas_gbs": by / cb / 1e6}))
PY
