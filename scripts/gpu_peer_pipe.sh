#!/bin/bash
# Pipelined cross-GPU prefix-hit epochs: GPU peer tests + the 2-rank one-GPU bench protocol.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/peer_tests.log 2>&1; echo "rc=$?" >> gpurun_out/peer_tests.log
GLMX_CHECK_ROTATIONS=14 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr=127.0.0.1 --master-port=29531 scripts/peer_pipeline_check.py > gpurun_out/peer_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/peer_pipe.log
for M in "" "--no-pipeline"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=29533 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline $M \
    > gpurun_out/bench_n2_pipe$M.json 2> gpurun_out/bench_n2_pipe$M.err
done
