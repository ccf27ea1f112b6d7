#!/bin/bash
# K1 at 65536 chunks (C2 graph, k=16): launch list of one chunk_build (all kernels, durations +
# DRAM bytes) and one --set full capture of the render+tokenize kernel with source.
mkdir -p gpurun_out
TAG=${TAG:-k1}
cat > /tmp/k1_one.py <<'PY'
import random, sys, os
sys.path.insert(0, os.getcwd())
import paper_2511_01633_b200 as glmx
g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
ret = glmx.Retriever(g, chunk_k=16, vocab=128256)
rnd = random.Random(65536)
nodes = [rnd.randrange(g.node_count()) for _ in range(65536)]
for _ in range(3):
    ret.chunk_build(nodes)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_launches.csv python /tmp/k1_one.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chunk_regular" -s 2 -c 1 \
  -o gpurun_out/${TAG}_re python /tmp/k1_one.py > gpurun_out/${TAG}_re_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_re.ncu-rep --page raw --csv > gpurun_out/${TAG}_re_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_re.ncu-rep --page source --csv --print-source sass -k regex:chunk_regular > gpurun_out/${TAG}_re_sass.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_re.ncu-rep --page source --csv --print-source sass -k regex:chunk_tokens_kernel > gpurun_out/${TAG}_tok_sass.csv 2>/dev/null
