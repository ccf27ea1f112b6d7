#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_retrieve_node.py -x -q > gpurun_out/retr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/retr_tests.log
timeout 900 python scripts/workload_scale.py 5000 100000 > gpurun_out/wl_scale.jsonl 2>&1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-standalone > gpurun_out/bench_$i.json 2>/dev/null; done
