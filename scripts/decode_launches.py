"""One decode batch (R=8, 4 steps) between cudaProfilerStart/Stop, for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_01633_b200 as glmx  # noqa: E402

cfg = glmx.ModelConfig(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256, seed=0)
model = glmx.Model(cfg, device=0)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
kv = glmx.KvCacheState(8192, 16, glmx.PRIORITY, device=0, n_layers=32, n_kv_heads=8,
                       head_dim=128, headroom_pages=2048)
eng = glmx.Engine(model, kv, max_requests=R, max_batch_tokens=R * 400, max_decode=16,
                  max_context=4096)
reqs = [glmx.Request([f"r{r}w{i}" for i in range(300)], [(0, 300, 3)], f"s{r}") for r in range(R)]
eng.prefill(reqs)
eng.decode([4] * R)
eng.prefill(reqs)
torch.cuda.cudart().cudaProfilerStart()
eng.decode([4] * R)
torch.cuda.cudart().cudaProfilerStop()
