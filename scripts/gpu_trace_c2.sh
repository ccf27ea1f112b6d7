#!/bin/bash
mkdir -p gpurun_out
GLMX_TRACE_SHAPES=profiles/r1_c2_attn_shapes.json:3 timeout 300 python scripts/attn_trace.py 0 0 0 --raw > gpurun_out/trace_c2_b3.txt 2>&1
