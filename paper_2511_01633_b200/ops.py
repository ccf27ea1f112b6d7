"""K2 (RoPE + KV append into the paged pool) on caller-owned device tensors
(glmx_rope_kv_append_run) — kernel-level face for parity tests and bandwidth sweeps; the engine
launches the same kernel inside its forward."""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib


def rope_kv_append(qkv, pos, slot, pool, q_out, n_heads, n_kv_heads, layer=0,
                   rope_theta=500000.0, reps=1, stream=None):
    """qkv [T][(H+2Hkv)*hd] bf16, pos int32 [T], slot int64 [T] (page*B + offset), pool
    [pages][L][2][Hkv][B][hd] bf16, q_out [T][H][hd] bf16.  Returns mean device ms per launch."""
    import torch

    T = qkv.shape[0]
    n_pages, L, _, Hkv, B, hd = pool.shape
    assert Hkv == n_kv_heads and qkv.shape[1] == (n_heads + 2 * n_kv_heads) * hd
    assert pos.dtype == torch.int32 and slot.dtype == torch.int64
    ms = C.c_float(0.0)
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    check(lib().glmx_rope_kv_append_run(qkv.data_ptr(), pos.data_ptr(), slot.data_ptr(), T,
                                        n_heads, n_kv_heads, hd, rope_theta, pool.data_ptr(), L,
                                        layer, B, q_out.data_ptr(), reps, s, C.byref(ms)))
    return ms.value


def kv_gather(pool, pages, layer, kv, out, impl=0, reps=1, stream=None):
    """K2 gather: out [len(pages)*B][Hkv][hd] <- pool[pages][layer][kv] (TMA-staged when impl=0).
    Returns the mean device ms per launch."""
    import torch

    n_pages, L, _, Hkv, B, hd = pool.shape
    ms = C.c_float(0.0)
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    arr = (C.c_int32 * max(1, len(pages)))(*[int(p) for p in pages])
    check(lib().glmx_kv_gather_run(pool.data_ptr(), n_pages, L, Hkv, B, hd, layer, kv, arr,
                                   len(pages), out.data_ptr(), impl, reps, s, C.byref(ms)))
    return ms.value

