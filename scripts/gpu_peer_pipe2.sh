#!/bin/bash
mkdir -p gpurun_out
for CAP in 224 160 128; do
GLMX_CHECK_CAPACITY=$CAP timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr=127.0.0.1 --master-port=29531 scripts/peer_pipeline_check.py > gpurun_out/peer_pipe_$CAP.log 2>&1; echo "rc=$?" >> gpurun_out/peer_pipe_$CAP.log
done
