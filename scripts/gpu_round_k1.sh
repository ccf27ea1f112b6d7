bash scripts/gpu_round.sh
TAG=k1final bash scripts/gpu_k1.sh > /dev/null 2>&1
tail -1 gpurun_out/k1final_kernels.jsonl
