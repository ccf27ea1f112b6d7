import sys, numpy as np
sys.path.insert(0, '.')
import paper_2511_01633_b200 as glmx
from oracle.decoder import Decoder, token_ids
def words(n, t="w"): return [f"{t}{i}" for i in range(n)]
cfg = glmx.ModelConfig(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab=128256)
model = glmx.Model(cfg, 0)
kv = glmx.KvCacheState(64, 16, 0, device=0, n_layers=2, n_kv_heads=8, head_dim=128, headroom_pages=64)
eng = glmx.Engine(model, kv, max_requests=4, max_batch_tokens=1024, max_decode=2, max_context=1024)
W = model.export_all()
p = words(150)
reqs = [glmx.Request(p, [(0, 40, 0), (40, 150, 3)], "a")]
reps, first, logits = eng.prefill(reqs, want_logits=True)
ids = token_ids(p, cfg.vocab)
for emu in (False, True):
    d = Decoder(cfg, W, emulate_bf16=emu)
    ref, _ = d.forward(ids)
    err = np.abs(logits[0]-ref)
    print("emulate", emu, "max err", err.max(), "mean", err.mean(), "p99.9", np.quantile(err, 0.999), "ref std", ref.std())
# tiny decode margins
cfg = glmx.TINY
model = glmx.Model(cfg, 0)
kv = glmx.KvCacheState(64, 16, 0, device=0, n_layers=cfg.n_layers, n_kv_heads=cfg.n_kv_heads, head_dim=128, headroom_pages=64)
eng = glmx.Engine(model, kv, max_requests=4, max_batch_tokens=512, max_decode=4, max_context=512)
prompt = words(37)
reqs = [glmx.Request(prompt, [(0, 16, 0), (16, 37, 3)], "s0"), glmx.Request(prompt[:33] + ["x", "y"], [(0, 35, 1)], "s1")]
reps, first, logits = eng.prefill(reqs, want_logits=True)
out, last = eng.decode([3, 2], want_logits=True)
d = Decoder(cfg, model.export_all())
ids = token_ids(reqs[0].tokens, cfg.vocab)
seq = [first[0]] + out[0]
lg, past = d.forward(ids)
for t in range(3):
    lg, past = d.forward([seq[t]], past=past)
    top = np.argsort(lg)[-3:]
    print("step", t, "gpu next", seq[t+1], "oracle top3", top, lg[top])
print("gpu last logits for req0 at 12638/4425:", last[0][12638], last[0][4425])
