"""How far do logits move from bf16 activation rounding alone? (CPU, numpy; no GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2511_01633_b200 as glmx
from oracle.decoder import Decoder, token_ids, bf16_round
cfg = glmx.ModelConfig(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab=128256)
rng = np.random.default_rng(0)
def w(*s): return bf16_round(rng.standard_normal(s, dtype=np.float32) * 0.02)
qkv = (32 + 16) * 128
W = {"embed": w(cfg.vocab, 4096), "final_norm": np.ones(4096, np.float32), "lm_head": w(cfg.vocab, 4096),
     "layers": [{"attn_norm": np.ones(4096, np.float32), "wqkv": w(qkv, 4096), "wo": w(4096, 4096),
                 "mlp_norm": np.ones(4096, np.float32), "w_gate_up": w(2 * 14336, 4096), "w_down": w(4096, 14336)} for _ in range(2)]}
ids = token_ids([f"w{i}" for i in range(150)], cfg.vocab)
t = time.time()
a, _ = Decoder(cfg, W).forward(ids)
b, _ = Decoder(cfg, W, emulate_bf16=True).forward(ids)
err = np.abs(a - b)
print(f"fp32 vs bf16-emulated: max {err.max():.4f} mean {err.mean():.4f} p99.9 {np.quantile(err, .999):.4f} std(logits) {a.std():.3f}  ({time.time()-t:.1f}s)")
print("within 2e-2+1e-2|ref|:", bool(np.all(err <= 2e-2 + 1e-2 * np.abs(a))))

# chaos floor: the bf16-emulating oracle against itself with small relative weight noise (the
# size of fp32 accumulation-order differences)
for eps, seed in ((1e-7, 1), (1e-7, 2), (1e-6, 1), (1e-6, 2), (4e-6, 1)):
    rng2 = np.random.default_rng(seed)
    Wp = dict(W, layers=[{k: ((v * (1 + eps * rng2.standard_normal(v.shape, dtype=np.float32)))
                              .astype(np.float32) if v.ndim == 2 else v) for k, v in l.items()}
                         for l in W["layers"]])
    c, _ = Decoder(cfg, Wp, emulate_bf16=True).forward(ids)
    e = np.abs(b - c)
    c32, _ = Decoder(cfg, Wp).forward(ids)
    print(f"eps {eps:g} seed {seed}: bf16-emulated vs perturbed: max {e.max():.4f} mean "
          f"{e.mean():.5f} in 2e-2/1e-2 {np.mean(e <= 2e-2 + 1e-2 * np.abs(b)):.5f}; "
          f"fp32 vs perturbed fp32: max {np.abs(a - c32).max():.2e}")
