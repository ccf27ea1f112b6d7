#!/bin/bash
# K1 kernel bench over prebuilt library variants (libglmx_*.so.tmp at the repo root)
mkdir -p gpurun_out
for f in libglmx_*.so.tmp; do
  for rep in 1 2; do
    GLMX_LIB=$PWD/$f timeout 300 python scripts/bench_kernels.py --skip K2 K2g K4 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$f', round(d['ms']*1000,1), 'us', round(d['hbm_frac'],3))"
  done
done
