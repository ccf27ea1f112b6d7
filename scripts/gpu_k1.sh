#!/bin/bash
# K1 check: GPU parity tests of the chunk builder, the kernel bench and the ncu captures.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${TAG:-k1}
timeout 900 python -m pytest tests/test_gpu_chunks.py tests/test_retrieve_node.py -q -x > gpurun_out/pytest_k1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1.log
timeout 300 python scripts/bench_kernels.py --skip K2 K2g K4 > gpurun_out/${TAG}_kernels.jsonl 2> gpurun_out/${TAG}_kernels.err
TAG=$TAG bash scripts/ncu_k1.sh
tail -3 gpurun_out/pytest_k1.log; cat gpurun_out/${TAG}_kernels.jsonl
