#!/bin/bash
# Round check: GPU tests, smoke, bench (+ reference arm), launch list of the timed step with DRAM
# bytes (ncu, profiler range = the timed rotations), traffic summary for bench.py.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
GLMX_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file gpurun_out/c2_step_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c2_step_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/c2_step_launches.csv --traffic gpurun_out/r1_c2_traffic.json > gpurun_out/c2_step_summary.txt 2>&1
cp gpurun_out/r1_c2_traffic.json profiles/r1_c2_traffic.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# K3 full ncu capture at the C5 shape (P = 8192, 8 requests) for profiles/
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn_tc -s 3 -c 1 \
    -o gpurun_out/attn_v3_p8192 python scripts/bench_attn.py --prefix 8192 --suffix 128 --batch 8 --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/attn_v3_p8192.ncu-rep --page raw --csv > gpurun_out/attn_v3_p8192_raw.csv 2>/dev/null
# N=2 protocol on the one GPU (gloo control plane): cross-GPU prefix hits through CUDA IPC + K4
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 8 --warmup 3 > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err
