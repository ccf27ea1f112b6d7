#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_retrieve_node.py tests/test_gpu_engine.py -x -q > gpurun_out/retr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/retr_tests.log
timeout 900 python scripts/workload_scale.py > gpurun_out/wl_scale.jsonl 2>&1
