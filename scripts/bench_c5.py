"""C5 long-context sweep (BASELINE.json configs[4]): vertex-chunk notebooks of P tokens cached in
the paged pool, then a reasoning prefill whose suffix is one new k-neighbour chunk + question.
Reports the K3 attention kernel's device time (CUDA events, mean of replays of the same staged
batch) and achieved TFLOP/s / GB/s against the measured peaks, for the tcgen05 kernel (default)
or the mma.sync baseline (GLMX_ATTN=mma).

usage: python scripts/bench_c5.py [--layers 32] [--batch 8] [--prefix 2048 8192 32768] [--k 16 64]
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.templates import TemplateSet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--prefix", type=int, nargs="+", default=[2048, 4096, 8192, 16384, 32768])
ap.add_argument("--k", type=int, nargs="+", default=[8, 16, 32, 64])
ap.add_argument("--replays", type=int, default=5)
ap.add_argument("--gemm-tune-tokens", type=int, default=12288,
                help="cuBLAS algorithm table up to this many batch tokens (0 = cublasGemmEx default)")
args = ap.parse_args()

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
cfg = glmx.ModelConfig(n_layers=args.layers, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256)
g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
model = glmx.Model(cfg, device=0)
if args.gemm_tune_tokens > 0:
    model.tune_gemms(args.gemm_tune_tokens)
max_ctx = max(args.prefix) + 4096
t = TemplateSet()
rows = []
for P in args.prefix:
    B = max(1, min(args.batch, (16384 * 16) // (P + 1024)))
    cap = B * (P + 2048) // 16 + 64
    # headroom: warm-up prefills of every k evict earlier notebooks; their pages are deferred-freed
    kv = glmx.KvCacheState(cap, 16, glmx.PRIORITY, device=0,
                           n_layers=cfg.n_layers, n_kv_heads=8, head_dim=128, headroom_pages=cap)
    eng = glmx.Engine(model, kv, max_requests=B, max_batch_tokens=max(8192, P + 2048),
                      max_decode=4, max_context=max_ctx)
    for k in args.k:
        ret = glmx.Retriever(g, chunk_k=k, vocab=0)
        rnd = random.Random(P * 100 + k)
        notebooks, last = [], []
        for b in range(B):
            nb = ""
            while len(nb.split()) < P - 80:
                nb += ret.chunk_build([rnd.randrange(g.node_count())]).texts[0] + "\n"
            notebooks.append(nb)
            # one fresh last chunk per replay: every measured prefill reuses the cached notebook
            # and computes a new suffix (chunk + question)
            last.append([ret.chunk_build([rnd.randrange(g.node_count())]).texts[0] + "\n"
                         for _ in range(args.replays + 1)])
        q = "Which item is linked from all of: v0000001; v0000002?"
        from paper_2511_01633_b200.workload import Call, GraphCoTWorkload, Session
        sess = [Session(f"c5_{P}_{k}_{b}", [0], q) for b in range(B)]
        warm_calls = [Call(sess[b], "reasoning", t.render_reasoning(q, notebooks[b]), "") for b in range(B)]
        meas_calls = [[Call(sess[b], "reasoning", t.render_reasoning(q, notebooks[b] + last[b][r]), "")
                       for b in range(B)] for r in range(args.replays + 1)]
        wl = GraphCoTWorkload.__new__(GraphCoTWorkload)
        wl.engine = eng
        wl.prefill(warm_calls[:1])
        for b in range(1, B):
            wl.prefill(warm_calls[b:b + 1])
        wl.prefill(meas_calls[0])  # warm-up of the measured shape
        eng.set_profiling(2)
        attn = fwd = flops = byts = 0.0
        for r in range(1, args.replays + 1):
            reps, _ = wl.prefill(meas_calls[r])
            tm = eng.last_timings()
            wk = eng.last_work()
            attn += tm["attention"]
            fwd += tm["forward"]
            flops += wk["attn_flops"]
            byts += wk["attn_bytes"]
        eng.set_profiling(0)
        attn /= args.replays
        fwd /= args.replays
        wk = {"attn_flops": flops / args.replays, "attn_bytes": byts / args.replays}
        tfl = wk["attn_flops"] / (attn * 1e-3) / 1e12
        gbs = wk["attn_bytes"] / (attn * 1e-3) / 1e9
        s = sum(r.computed_tokens + r.tail_tokens for r in reps) / B
        cached = sum(r.cached_tokens for r in reps) / B
        row = {"prefix": P, "k": k, "batch": B, "suffix_tokens": s, "cached_tokens": cached,
               "attn_ms_per_forward": attn, "attn_ms_per_layer": attn / cfg.n_layers,
               "attn_tflops": tfl,
               # timed inside the forward (GEMMs interleaved, power-capped clocks): sustained peak
               "tensor_frac": tfl / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
               "attn_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
               "intensity": wk["attn_flops"] / wk["attn_bytes"], "forward_ms": fwd,
               # effective prompt tokens/s of a 32-layer forward, extrapolated from n_layers
               "prefill_tokens_per_s_32l": sum(r.cached_tokens + r.computed_tokens + r.tail_tokens
                                               for r in reps) / (fwd * 1e-3 * 32 / cfg.n_layers),
               "attn_share": attn / fwd,
               "impl": "tc"}
        rows.append(row)
        print(json.dumps(row), flush=True)
    del eng, kv
