"""Decode step cost: wall per greedy step vs device forward time (CUDA events on the engine
stream) for R requests at the Llama-3-8B shape — is decode launch-bound on the host?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402

cfg = glmx.ModelConfig(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256, seed=0)
model = glmx.Model(cfg, device=0)
for R in (8, 64, 128):
    kv = glmx.KvCacheState(8192, 16, glmx.PRIORITY, device=0, n_layers=32, n_kv_heads=8,
                           head_dim=128, headroom_pages=2048)
    eng = glmx.Engine(model, kv, max_requests=R, max_batch_tokens=R * 400, max_decode=16,
                      max_context=4096)
    reqs = [glmx.Request([f"r{r}w{i}" for i in range(300)], [(0, 300, 3)], f"s{r}") for r in range(R)]
    eng.prefill(reqs)
    eng.set_profiling(1)
    for steps in (1, 16):
        eng.prefill(reqs)  # restage the batch (all cached now)
        t0 = time.perf_counter()
        eng.decode([steps] * R)
        wall = time.perf_counter() - t0
        tm = eng.last_timings()
        print(f"R={R} steps={steps}: wall {1e3 * wall / steps:.2f} ms/step, device forward "
              f"{tm['forward'] / steps:.2f} ms/step")
    del eng, kv
