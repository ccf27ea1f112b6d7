#!/bin/bash
# final ncu --set full summaries: K3d (decode attention, 64 x 1500 contexts), K2 inside the C2 step
# (head-group version), K1 render+tokenize (65536 chunks)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:decode_attn -s 2 -c 1 -o gpurun_out/k3d_final \
  python scripts/bench_attn.py --impl 2 --prefix 1500 --suffix 1 --batch 64 --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/k3d_final.ncu-rep --page raw --csv > gpurun_out/k3d_final_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:rope_kv_append -s 100 -c 1 -o gpurun_out/k2_final \
  python bench.py --no-cpu-baseline --no-standalone --steps 2 --warmup 3 --decode-steps 0 > /dev/null 2>&1
ncu -i gpurun_out/k2_final.ncu-rep --page raw --csv > gpurun_out/k2_final_raw.csv 2>/dev/null
sed -i 's/-k regex:"chunk_render_emit" -s 1 -c 1/-k regex:"chunk_render_emit" -s 1 -c 1/' scripts/ncu_k1.sh
bash scripts/ncu_k1.sh
