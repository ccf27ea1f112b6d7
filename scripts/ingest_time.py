"""Graph ingest time: the 100k-node / 800k-edge power-law JSONL, host-only build vs
device build (threaded parse + entries on the host, CSRs and weights on the GPU)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402

g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=-1)
path = "/tmp/ingest_100k.jsonl"
g.save(path)
glmx.PropertyGraph.load(path, device=0)  # CUDA context / module load outside the timing
for dev in (-1, 0):
    t0 = time.perf_counter()
    h = glmx.PropertyGraph.load(path, device=dev)
    dt = time.perf_counter() - t0
    print(json.dumps({"nodes": h.node_count(), "edges": h.edge_count(),
                      "build": "host CSR" if dev < 0 else "GPU CSR", "seconds": dt}), flush=True)
