"""Where the C2 rotation's wall time goes on the host (e2e vs device forward): next_calls /
pack (Python), the prefill C-ABI call (bookkeeping + H2D + forward + D2H), advance (notebook
updates, K1 join).  Same setup as bench.py."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.workload import GraphCoTWorkload  # noqa: E402

cfg = glmx.ModelConfig(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256, seed=0)
g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
model = glmx.Model(cfg, device=0)
kv = glmx.KvCacheState(16384, 16, glmx.PRIORITY, device=0, n_layers=32, n_kv_heads=8,
                       head_dim=128, headroom_pages=4096)
eng = glmx.Engine(model, kv, max_requests=64, max_batch_tokens=64 * 1024, max_decode=8,
                  max_context=8192)
wl = GraphCoTWorkload(eng, ret, n_queries=64 * 3, lanes=64, seed=0, question_pool=96,
                      node_index=glmx.NodeIndex(g))
eng.set_profiling(1)
for r in range(11):
    t0 = time.perf_counter()
    calls = wl.next_calls()
    t1 = time.perf_counter()
    packed = wl.pack(calls)
    t2 = time.perf_counter()
    reps, first = wl.prefill(calls, packed)
    t3 = time.perf_counter()
    wl.advance(calls, reps, first)
    t4 = time.perf_counter()
    tm = eng.last_timings()
    print(f"rot {r}: next_calls {1e3*(t1-t0):6.2f} pack {1e3*(t2-t1):6.2f} prefill {1e3*(t3-t2):7.2f} "
          f"(device fwd {tm['forward']:7.2f}, h2d {tm.get('h2d', 0):5.2f}) advance {1e3*(t4-t3):6.2f} ms")
