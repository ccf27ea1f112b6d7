"""Merged (deferred) decode vs two separate decodes: device time of the decode forwards."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402

cfg = glmx.ModelConfig(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256, seed=0)
model = glmx.Model(cfg, device=0)
R = 64
kv = glmx.KvCacheState(16384, 16, glmx.PRIORITY, device=0, n_layers=32, n_kv_heads=8,
                       head_dim=128, headroom_pages=4096)
eng = glmx.Engine(model, kv, max_requests=R, max_batch_tokens=R * 400, max_decode=16,
                  max_context=4096)
A = [glmx.Request([f"a{r}w{i}" for i in range(300)], [(0, 300, 3)], f"a{r}") for r in range(R)]
Bq = [glmx.Request([f"b{r}w{i}" for i in range(300)], [(0, 300, 3)], f"b{r}") for r in range(R)]
eng.set_profiling(1)
for it in range(3):
    for steps in (1, 4):
        eng.prefill(A)
        eng.decode_async([steps] * R)
        eng.decode_collect()
        ta = eng.last_timings()["forward"]
        eng.prefill(Bq)
        eng.decode_async([steps] * R)
        eng.decode_collect()
        tb = eng.last_timings()["forward"]
        eng.prefill(A)
        eng.decode_defer([steps] * R)
        eng.prefill(Bq)
        eng.decode_async([steps] * R)
        cur, prev = eng.decode_collect()
        tm = eng.last_timings()["forward"]
        print(f"steps={steps}: separate {ta:.2f} + {tb:.2f} = {ta + tb:.2f} ms, merged {tm:.2f} ms")
