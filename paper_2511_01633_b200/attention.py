"""K3 paged prefill attention on caller-owned device tensors (glmx_attention_run).

The engine calls the same kernel inside its forward; this face exists for kernel-level parity
tests and attention sweeps (long-context configuration C5).  Tensors are torch CUDA tensors used
only as device memory: q/o [rows][H][hd] bf16, pool [pages][L][2][Hkv][B][hd] bf16.
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib

TC = 0   # tcgen05 / TMEM / TMA kernel (the product path)
DECODE = 2  # CUDA-core flash-decoding kernel for one-token rows (the engine's decode steps)


def _i32(xs):
    arr = (C.c_int32 * max(1, len(xs)))(*[int(x) for x in xs])
    return arr


def paged_attention(q, o, pool, q_start, q_len, ctx_len, block_table, layer=0, impl=TC,
                    reps=1, stream=None):
    """Run K3 over n_req requests; returns the mean device ms per launch.

    q_start/q_len/ctx_len: per-request ints; block_table: list of page lists (padded here)."""
    import torch

    assert q.dtype == torch.bfloat16 and o.dtype == torch.bfloat16 and pool.dtype == torch.bfloat16
    assert q.is_cuda and o.is_cuda and pool.is_cuda and q.is_contiguous() and o.is_contiguous()
    n_pages, L, two, Hkv, B, hd = pool.shape
    assert two == 2 and q.shape[2] == hd
    rows, H = q.shape[0], q.shape[1]
    n = len(q_len)
    stride = max(1, max(len(b) for b in block_table))
    bt = []
    for b in block_table:
        bt.extend(list(b) + [0] * (stride - len(b)))
    ms = C.c_float(0.0)
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    check(lib().glmx_attention_run(impl, q.data_ptr(), o.data_ptr(), rows, H, Hkv, hd,
                                   pool.data_ptr(), n_pages, L, layer, B, n, _i32(q_start),
                                   _i32(q_len), _i32(ctx_len), _i32(bt), stride, reps, s,
                                   C.byref(ms)))
    return ms.value


def schedule(work, q_len, ctx_len, n_kv_heads=8, tokens_per_item=64, n_sm=148, pair=True):
    """K3's stream-K schedule (host C++ build_attn_schedule) for inspection/tests.

    work: list of (request, first token).  Returns dict(pieces=[(item, j0, j1, part)],
    partners=[(item or -1, j0, j1, part)] (one per piece), cta_off=[...],
    combine=[(item, part0, n_part)], grid, n_partials, total_tiles)."""
    n_items = len(work) * n_kv_heads
    flat = [int(v) for xy in work for v in xy]
    pieces = (C.c_int32 * (4 * (n_items + n_sm)))()
    cta = (C.c_int32 * (n_sm + 1))()
    comb = (C.c_int32 * (4 * n_sm))()
    partners = (C.c_int32 * (4 * (n_items + n_sm)))() if pair else None
    cnt = (C.c_int64 * 5)()
    check(lib().glmx_attn_schedule(_i32(flat), len(work), n_kv_heads, _i32(q_len), _i32(ctx_len),
                                   tokens_per_item, n_sm, pieces, cta, comb, partners, cnt))
    n_p, grid, n_c, n_part, total = list(cnt)
    return {"pieces": [tuple(pieces[4 * i:4 * i + 4]) for i in range(n_p)],
            "partners": [tuple(partners[4 * i:4 * i + 4]) if pair else (-1, 0, 0, -1)
                         for i in range(n_p)],
            "cta_off": list(cta[:grid + 1]),
            "combine": [tuple(comb[4 * i:4 * i + 3]) for i in range(n_c)],
            "grid": grid, "n_partials": n_part, "total_tiles": total}
