"""K3 kernel-level sweep (C5 long-context shapes): B requests, each with a P-token cached prefix
and an s-token suffix, Llama-3-8B attention geometry (32 q / 8 kv heads, hd 128, 16-token pages).
Times glmx_attention_run (CUDA events, mean of `reps` back-to-back launches after warm-up) and
reports TFLOP/s against the measured bf16 peak and GB/s (algorithmic KV bytes) against HBM.

usage: python scripts/bench_attn.py [--impl 0|1] [--prefix 2048 8192 32768] [--suffix 128]
                                    [--batch 8] [--reps 20]
"""
import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_01633_b200.attention as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--impl", type=int, default=0)
ap.add_argument("--prefix", type=int, nargs="+", default=[2048, 8192, 32768])
ap.add_argument("--suffix", type=int, nargs="+", default=[128])
ap.add_argument("--batch", type=int, nargs="+", default=[8])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--check", action="store_true", help="compare against the fp32 reference")
ap.add_argument("--shapes", default=None,
                help="JSON list of batches [[ctx, q_len], ...] (scripts/c2_attn_shapes.py)")
args = ap.parse_args()

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
H, Hkv, hd, B = 32, 8, 128, 16


def run_batch(reqs, tag):
    """One ragged batch: reqs = [(ctx, q_len)]; returns the JSON row."""
    pages_of = [(c + B - 1) // B for c, _ in reqs]
    n_pages = sum(pages_of)
    pool = torch.empty((n_pages, args.layers, 2, Hkv, B, hd), dtype=torch.bfloat16,
                       device="cuda").normal_()
    rows = sum(q for _, q in reqs)
    q = torch.empty((rows, H, hd), dtype=torch.bfloat16, device="cuda").normal_()
    o = torch.empty_like(q)
    perm = list(range(n_pages))
    random.Random(rows).shuffle(perm)
    bt, qs, ql, cl = [], [], [], []
    p = r = 0
    for (c, n), k in zip(reqs, pages_of):
        bt.append(perm[p:p + k])
        p += k
        qs.append(r)
        ql.append(n)
        cl.append(c)
        r += n
    A.paged_attention(q, o, pool, qs, ql, cl, bt, impl=args.impl, reps=3)
    ms = A.paged_attention(q, o, pool, qs, ql, cl, bt, impl=args.impl, reps=args.reps)
    flops = sum(4.0 * H * hd * (c - n + t + 1) for c, n in reqs for t in range(n))
    kv_bytes = sum(c * Hkv * hd * 2 * 2 + 2 * n * H * hd * 2 for c, n in reqs)
    return {"impl": "tc" if args.impl == 0 else "decode", "batch": tag, "requests": len(reqs),
            "ms": ms, "tflops": flops / ms / 1e9, "tensor_frac": flops / ms / 1e9 / peaks["bf16_tflops"],
            "gbs": kv_bytes / ms / 1e6, "hbm_frac": kv_bytes / ms / 1e6 / peaks["hbm_gbs"],
            "intensity": flops / kv_bytes}


if args.shapes:
    tot_ms = 0.0
    for i, reqs in enumerate(json.load(open(args.shapes))):
        row = run_batch([tuple(x) for x in reqs], i)
        tot_ms += row["ms"]
        print(json.dumps(row), flush=True)
    print(json.dumps({"total_ms_per_layer": tot_ms}))
    sys.exit(0)

for P in args.prefix:
    for s in args.suffix:
        for nb in args.batch:
            ctx = P + s
            pages_per = (ctx + B - 1) // B
            n_pages = nb * pages_per
            pool = torch.empty((n_pages, args.layers, 2, Hkv, B, hd), dtype=torch.bfloat16,
                               device="cuda").normal_()
            q = torch.empty((nb * s, H, hd), dtype=torch.bfloat16, device="cuda").normal_()
            o = torch.empty_like(q)
            perm = list(range(n_pages))
            random.Random(P + s).shuffle(perm)
            bt = [perm[i * pages_per:(i + 1) * pages_per] for i in range(nb)]
            qs = [i * s for i in range(nb)]
            ql = [s] * nb
            cl = [ctx] * nb
            A.paged_attention(q, o, pool, qs, ql, cl, bt, impl=args.impl, reps=3)
            ms = A.paged_attention(q, o, pool, qs, ql, cl, bt, impl=args.impl, reps=args.reps)
            flops = nb * sum(4.0 * H * hd * (P + t + 1) for t in range(s))
            kv_bytes = nb * (ctx * Hkv * hd * 2 * 2 + 2 * s * H * hd * 2)
            row = {"impl": "tc" if args.impl == 0 else "decode", "prefix": P, "suffix": s,
                   "batch": nb, "ms": ms, "tflops": flops / ms / 1e9,
                   "tensor_frac": flops / ms / 1e9 / peaks["bf16_tflops"],
                   "gbs": kv_bytes / ms / 1e6, "hbm_frac": kv_bytes / ms / 1e6 / peaks["hbm_gbs"],
                   "intensity": flops / kv_bytes}
            if args.check:
                sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
                from torch_refs import reference_attention
                ref = reference_attention(q, pool, qs, ql, cl, bt)
                err = (o.float() - ref).abs()
                row["max_err"] = err.max().item()
                row["in_tol"] = bool((err <= 2e-2 + 1e-2 * ref.abs()).all().item())
            print(json.dumps(row), flush=True)
            del pool, q, o
            torch.cuda.empty_cache()
