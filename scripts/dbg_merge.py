import sys, os
sys.path.insert(0, os.getcwd())
import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200.workload import GraphCoTWorkload, count_tokens
cfg = glmx.ModelConfig(n_layers=4, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab=128256, seed=0)
g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
model = glmx.Model(cfg, device=0)
kv = glmx.KvCacheState(16384, 16, glmx.PRIORITY, device=0, n_layers=4, n_kv_heads=8, head_dim=128, headroom_pages=4096)
eng = glmx.Engine(model, kv, max_requests=64, max_batch_tokens=64 * 1024, max_decode=8, max_context=8192)
wl = GraphCoTWorkload(eng, ret, n_queries=64 * 6, lanes=64, seed=0, question_pool=192)
for merge in (False, True):
    eng.set_profiling(1)
    for r in wl.rotations_with_decode(8, 8, merge=merge):
        print(merge, "rot steps total", r.decoded_tokens, "collected", r.decode_collected, "dec ms %.2f" % (eng.last_timings()["forward"] if r.decode_collected else -1))
    print([ (k, max((len(c) for c in v), default=0)) for k, v in wl.decode_log])
