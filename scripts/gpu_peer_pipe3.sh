#!/bin/bash
mkdir -p gpurun_out
GLMX_CHECK_CAPACITY=160 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr=127.0.0.1 --master-port=29531 scripts/peer_pipeline_check.py > gpurun_out/peer_pipe3.log 2>&1; echo "rc=$?" >> gpurun_out/peer_pipe3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=29533 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
