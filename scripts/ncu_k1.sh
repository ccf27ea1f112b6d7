#!/bin/bash
mkdir -p gpurun_out
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chunk_render_emit" -s 1 -c 1 \
  -o gpurun_out/k1_re python /tmp/k1_one.py > gpurun_out/k1_re_ncu.log 2>&1
ncu -i gpurun_out/k1_re.ncu-rep --page raw --csv > gpurun_out/k1_re_raw.csv 2>/dev/null
ncu -i gpurun_out/k1_re.ncu-rep --page source --csv --print-source sass -k regex:chunk_render_emit > gpurun_out/k1_re_sass.csv 2>/dev/null
ncu -i gpurun_out/k1_re.ncu-rep --page details --csv > gpurun_out/k1_re_details.csv 2>/dev/null
