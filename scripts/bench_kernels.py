"""HBM-bound kernels of the hot path against the measured copy bandwidth (MEASURED_PEAKS.json):

  K2  rope_kv_append  — fused RoPE + paged KV append (glmx_rope_kv_append_run), T tokens of the
                        Llama-3-8B shape; algorithmic bytes/token = read qkv 12288 + write q 8192
                        + write K,V 4096 = 24576 B
  K4  pool_copy       — whole-page copies inside one pool (glmx_pool_copy), 2 MiB pages;
                        2 x page bytes per page (read + write)
  K1  chunk_build     — vertex-chunk assembly over a batch of nodes of the 100k-node graph, k=16;
                        bytes = CSR rows + neighbour (idx, weight) pairs + entry bytes read +
                        chunk bytes + 20 B/token written (approximate: undirected degree from
                        glmx_graph_degree)

usage: python scripts/bench_kernels.py [--reps 20]
"""
import argparse
import ctypes as C
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200._lib import check, lib  # noqa: E402
from paper_2511_01633_b200.ops import rope_kv_append  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--skip", nargs="*", default=[])
ap.add_argument("--k2-tokens", type=int, nargs="+", default=[520, 2750, 4965, 16384])
args = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM = peaks["hbm_gbs"]


def emit(row):
    row["hbm_frac"] = row["gbs"] / HBM
    print(json.dumps(row), flush=True)


H, Hkv, hd, B, L = 32, 8, 128, 16, 32
if "K2" not in args.skip:
    for T in args.k2_tokens:
        n_pages = (T + B - 1) // B + 8
        pool = torch.zeros((n_pages, L, 2, Hkv, B, hd), dtype=torch.bfloat16, device="cuda")
        qkv = torch.randn((T, (H + 2 * Hkv) * hd), device="cuda").to(torch.bfloat16)
        pos = torch.randint(0, 8192, (T,), dtype=torch.int32, device="cuda")
        perm = torch.randperm(n_pages)[: (T + B - 1) // B]
        slot = torch.tensor([int(perm[t // B]) * B + t % B for t in range(T)],
                            dtype=torch.int64, device="cuda")
        q_out = torch.empty((T, H, hd), dtype=torch.bfloat16, device="cuda")
        rope_kv_append(qkv, pos, slot, pool, q_out, H, Hkv, layer=5, reps=3)
        ms = rope_kv_append(qkv, pos, slot, pool, q_out, H, Hkv, layer=5, reps=args.reps)
        by = T * ((H + 2 * Hkv) * hd * 2 + H * hd * 2 + 2 * Hkv * hd * 2)
        emit({"kernel": "K2 rope_kv_append", "tokens": T, "ms": ms, "bytes": by,
              "gbs": by / ms / 1e6})
        del pool, qkv, q_out
        torch.cuda.empty_cache()

if "K2g" not in args.skip:
    from paper_2511_01633_b200.ops import kv_gather
    for n, impl in ((512, 0), (4096, 0), (16384, 0), (4096, 1)):
        pool = torch.zeros((n + 8, 4, 2, Hkv, B, hd), dtype=torch.bfloat16, device="cuda")
        out = torch.empty((n * B, Hkv, hd), dtype=torch.bfloat16, device="cuda")
        pages = torch.randperm(n + 8)[:n].tolist()
        kv_gather(pool, pages, 1, 0, out, impl=impl, reps=3)
        ms = kv_gather(pool, pages, 1, 0, out, impl=impl, reps=args.reps)
        by = 2 * n * Hkv * B * hd * 2
        emit({"kernel": "K2 kv_gather (" + ("TMA-staged" if impl == 0 else "scalar") + ")",
              "pages": n, "ms": ms, "bytes": by, "gbs": by / ms / 1e6})
        del pool, out
        torch.cuda.empty_cache()

if "K4" not in args.skip:
    for n in [64, 1024]:
        kv = glmx.KvCacheState(2 * n + 16, 16, glmx.PRIORITY, device=0, n_layers=L, n_kv_heads=Hkv,
                               head_dim=hd, headroom_pages=16)
        src = list(range(n))
        dst = list(range(n, 2 * n))
        random.Random(n).shuffle(dst)
        s_arr = (C.c_int32 * n)(*src)
        d_arr = (C.c_int32 * n)(*dst)
        stream = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            check(lib().glmx_pool_copy(kv.h, kv.h, s_arr, d_arr, n, stream))
        tot = 0.0
        for _ in range(args.reps):
            check(lib().glmx_pool_copy(kv.h, kv.h, s_arr, d_arr, n, stream))
            tot += lib().glmx_pool_last_copy_ms(kv.h)
        ms = tot / args.reps
        page = lib().glmx_kv_page_bytes(kv.h)
        by = 2 * n * page
        emit({"kernel": "K4 pool_copy (local)", "pages": n, "page_bytes": page, "ms": ms,
              "bytes": by, "gbs": by / ms / 1e6})
        kv.close()

if "K1" not in args.skip:
    g = glmx.PropertyGraph.synth_powerlaw(100000, 8, seed=0, device=0)
    ret = glmx.Retriever(g, chunk_k=16, vocab=128256)
    for n in [64, 4096, 65536]:
        rnd = random.Random(n)
        nodes = [rnd.randrange(g.node_count()) for _ in range(n)]
        ret.chunk_build(nodes)
        ms_list = []
        for _ in range(max(3, args.reps // 4)):
            cb = ret.chunk_build(nodes)
            ms_list.append(cb.kernel_ms)
        ms = sorted(ms_list)[len(ms_list) // 2]
        out_bytes = sum(len(t.encode()) for t in cb.texts)
        tokens = sum(len(x) for x in cb.token_spans)
        deg = sum(g.total_degree(i) for i in nodes)
        by = 8 * n + 8 * deg + 2 * out_bytes + 20 * tokens
        emit({"kernel": "K1 chunk_build (select+scan+render+tokenize)", "chunks": n, "ms": ms,
              "bytes": by, "gbs": by / ms / 1e6, "out_bytes": out_bytes, "tokens": tokens,
              "note": "ms spans the 4 launches + one host sync for the output size"})
