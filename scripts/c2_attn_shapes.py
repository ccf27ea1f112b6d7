"""Dump the per-rotation attention shapes (ctx_len, q_len) of the C2 Graph-CoT workload (same
setup as bench.py, 1-layer model: cache decisions do not depend on the model) to a JSON file for
scripts/bench_attn.py --shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.workload import GraphCoTWorkload  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c2_shapes.json"
rot = int(sys.argv[2]) if len(sys.argv) > 2 else 11
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # untimed rotations first (bench: 64 + 3)
cfg = glmx.ModelConfig(n_layers=1, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256, seed=0)
g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
model = glmx.Model(cfg, device=0)
kv = glmx.KvCacheState(16384, 16, glmx.PRIORITY, device=0, n_layers=1, n_kv_heads=8, head_dim=128,
                       headroom_pages=4096)
eng = glmx.Engine(model, kv, max_requests=64, max_batch_tokens=64 * 1024, max_decode=8,
                  max_context=8192)
# the bench's workload: RetrieveNode through the index, 22% repeated questions
wl = GraphCoTWorkload(eng, ret, n_queries=64 * ((warm + rot) // 6 + 2), lanes=64, seed=0,
                      node_index=glmx.NodeIndex(g), repeat_frac=0.22)
for _ in range(warm):
    calls = wl.next_calls()
    reps, first = wl.prefill(calls)
    wl.advance(calls, reps, first)
batches = []
for _ in range(rot):
    calls = wl.next_calls()
    reps, first = wl.prefill(calls)
    wl.advance(calls, reps, first)
    b = []
    for r in reps:
        ctx = r.cached_tokens + r.computed_tokens + r.tail_tokens
        b.append((ctx, max(1, r.computed_tokens + r.tail_tokens)))
    batches.append(b)
json.dump(batches, open(out, "w"))
for b in batches:
    print(len(b), "calls, mean ctx", sum(c for c, _ in b) / len(b), "mean q", sum(q for _, q in b) / len(b))
