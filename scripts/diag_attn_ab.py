"""A/B: tcgen05 attention vs the mma.sync baseline inside the engine (same batch, same weights)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from oracle.decoder import Decoder, token_ids  # noqa: E402


def words(n, t="w"):
    return [f"{t}{i}" for i in range(n)]


def run(cfg, reqs, impl, decode=None):
    os.environ["GLMX_ATTN"] = impl
    model = glmx.Model(cfg, 0)
    kv = glmx.KvCacheState(4096, 16, 0, device=0, n_layers=cfg.n_layers, n_kv_heads=cfg.n_kv_heads,
                           head_dim=128, headroom_pages=512)
    eng = glmx.Engine(model, kv, max_requests=16, max_batch_tokens=8192, max_decode=8,
                      max_context=8192)
    t = time.time()
    reps, first, logits = eng.prefill(reqs, want_logits=True)
    out = eng.decode(decode) if decode else None
    return model, logits, first, out, time.time() - t


for name, cfg in [("tiny", glmx.TINY),
                  ("8b-2L", glmx.ModelConfig(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8,
                                             head_dim=128, d_ff=14336, vocab=128256))]:
    p = words(900)
    reqs = [glmx.Request(p[:700], [(0, 40, 0), (40, 700, 3)], "a"),
            glmx.Request(p[:520] + words(260, "y"), [(0, 780, 1)], "b"),  # 512 cached
            glmx.Request(words(3, "z"), [(0, 3, 3)], "c"),
            glmx.Request(p[:129], [(0, 129, 2)], "d")]
    m1, l_tc, f_tc, o_tc, t1 = run(cfg, reqs, "tc", [5, 5, 5, 5])
    m2, l_mma, f_mma, o_mma, t2 = run(cfg, reqs, "mma", [5, 5, 5, 5])
    d = np.abs(l_tc - l_mma)
    print(f"{name}: tc vs mma logits max {d.max():.5f} mean {d.mean():.6f}; first tc {f_tc} "
          f"mma {f_mma}; decode equal {o_tc == o_mma}", flush=True)
    if name == "tiny":
        dec = Decoder(cfg, m1.export_all())
        for i, r in enumerate(reqs):
            ref, _ = dec.forward(token_ids(r.tokens, cfg.vocab))
            e = np.abs(l_tc[i] - ref)
            print(f"  req {i} tc vs fp32 oracle: max {e.max():.5f} within tol "
                  f"{bool(np.all(e <= 2e-2 + 1e-2 * np.abs(ref)))}")
            dec.check_greedy(token_ids(r.tokens, cfg.vocab), [f_tc[i]] + o_tc[i])
        print("  greedy tc vs oracle ok")
