"""Random-init Llama-style decoder + the prefill/decode engine over the paged KV pool.

The engine call replaces the reference's cost line (orchestrator.cpp:131-132,
span = c_prefill*computed + c_decode*tokens_out) with a real forward: bookkeeping prefill in
request order, one batched layer-synchronous forward, greedy first token.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .kvcache import KvCacheState, PrefillReport, pack_tiers, pack_tokens


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    init_std: float = 0.02
    seed: int = 0

    def to_c(self):
        return _lib.ModelConfigC(self.n_layers, self.d_model, self.n_heads, self.n_kv_heads,
                                 self.head_dim, self.d_ff, self.vocab, self.rope_theta,
                                 self.norm_eps, self.init_std, self.seed)

    def kv_bytes_per_token(self):
        return self.n_layers * 2 * self.n_kv_heads * self.head_dim * 2


# C1 tiny decoder; C2/C5 Llama-3-8B shape.
TINY = ModelConfig(n_layers=2, d_model=512, n_heads=4, n_kv_heads=2, head_dim=128, d_ff=1024,
                   vocab=32000)
LLAMA3_8B = ModelConfig(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                        d_ff=14336, vocab=128256)

WEIGHTS = {"embed": 0, "attn_norm": 1, "wqkv": 2, "wo": 3, "mlp_norm": 4, "w_gate_up": 5,
           "w_down": 6, "final_norm": 7, "lm_head": 8}


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


class Model:
    def __init__(self, cfg: ModelConfig, device=0):
        self.cfg = cfg
        self.device = device
        h = C.c_void_p()
        c = cfg.to_c()
        check(lib().glmx_model_create(C.byref(c), device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().glmx_model_destroy(self.h)
            self.h = None

    __del__ = _lib.safe_del

    def tune_gemms(self, max_tokens: int) -> int:
        """Pick cuBLAS algorithms for the per-layer projections per M bucket up to max_tokens
        (glmx_model_tune_gemms); seconds of device time, call before any engine work. Returns
        the number of buckets where a candidate beat the default cublasGemmEx choice."""
        n = C.c_int32()
        check(lib().glmx_model_tune_gemms(self.h, int(max_tokens), C.byref(n)))
        return n.value

    def export(self, name, layer=0, shape=None) -> np.ndarray:
        """bf16 weights as float32 (for the CPU oracle)."""
        c = self.cfg
        qkv = (c.n_heads + 2 * c.n_kv_heads) * c.head_dim
        shapes = {"embed": (c.vocab, c.d_model), "attn_norm": (c.d_model,),
                  "wqkv": (qkv, c.d_model), "wo": (c.d_model, c.n_heads * c.head_dim),
                  "mlp_norm": (c.d_model,), "w_gate_up": (2 * c.d_ff, c.d_model),
                  "w_down": (c.d_model, c.d_ff), "final_norm": (c.d_model,),
                  "lm_head": (c.vocab, c.d_model)}
        shp = shapes[name]
        n = int(np.prod(shp))
        buf = np.empty(n, dtype=np.uint16)
        check(lib().glmx_model_export_weight(self.h, WEIGHTS[name], layer,
                                             buf.ctypes.data_as(C.POINTER(C.c_uint16)), n))
        return bf16_to_f32(buf).reshape(shp)

    def export_all(self):
        w = {"embed": self.export("embed"), "final_norm": self.export("final_norm"),
             "lm_head": self.export("lm_head"), "layers": []}
        for l in range(self.cfg.n_layers):
            w["layers"].append({k: self.export(k, l) for k in
                                ("attn_norm", "wqkv", "wo", "mlp_norm", "w_gate_up", "w_down")})
        return w


@dataclass
class Request:
    tokens: list          # list[str]
    tiers: list           # [(begin, end, tier)]
    session: str


class Engine:
    def __init__(self, model: Model, kv: KvCacheState, max_requests=64, max_batch_tokens=8192,
                 max_decode=64, max_context=8192):
        self.model = model
        self.kv = kv
        cfg = _lib.EngineConfig(max_requests, max_batch_tokens, max_decode, max_context)
        h = C.c_void_p()
        check(lib().glmx_engine_create(model.h, kv.h, C.byref(cfg), C.byref(h)))
        self.h = h
        self.max_requests = max_requests
        self.max_decode = max_decode
        self._keep = None

    def close(self):
        if getattr(self, "h", None):
            lib().glmx_engine_destroy(self.h)
            self.h = None

    __del__ = _lib.safe_del

    def set_profiling(self, on=True):
        lib().glmx_engine_set_profiling(self.h, int(on))

    def set_reuse(self, on=True):
        """KV reuse on/off (A/B): off recomputes cache hits into scratch pages."""
        lib().glmx_engine_set_reuse(self.h, int(on))

    @staticmethod
    def pack_requests(requests):
        n = len(requests)
        arr = (_lib.RequestC * max(1, n))()
        keep = []
        for i, r in enumerate(requests):
            blob, offs = pack_tokens(r.tokens)
            tarr = pack_tiers(r.tiers)
            sb = r.session.encode()
            keep += [blob, offs, tarr, sb]
            arr[i].tok_bytes = blob
            arr[i].tok_offsets = offs
            arr[i].n_tok = len(r.tokens)
            arr[i].tiers = tarr
            arr[i].n_tiers = len(r.tiers)
            arr[i].session = sb
        return arr, keep

    def prefill(self, requests, want_logits=False, packed=None):
        """Returns (reports, first_tokens[, logits])."""
        n = len(requests) if packed is None else packed[2]
        arr, keep = (self.pack_requests(requests) if packed is None else packed[:2])
        reps = (_lib.PrefillReportC * max(1, n))()
        first = (C.c_int32 * max(1, n))()
        logits = None
        lp = None
        if want_logits:
            logits = np.zeros((n, self.model.cfg.vocab), dtype=np.float32)
            lp = logits.ctypes.data_as(_lib.f32p)
        check(lib().glmx_engine_prefill(self.h, n, arr, reps, first, lp))
        out = [PrefillReport(reps[i].cached_tokens, reps[i].computed_tokens, reps[i].tail_tokens)
               for i in range(n)]
        toks = [first[i] for i in range(n)]
        return (out, toks, logits) if want_logits else (out, toks)

    def decode(self, steps, want_logits=False):
        n = len(steps)
        st = (C.c_uint32 * max(1, n))(*steps)
        m = max(steps) if steps else 0
        out = (C.c_int32 * max(1, n * m))()
        logits = None
        lp = None
        if want_logits:
            logits = np.zeros((n, self.model.cfg.vocab), dtype=np.float32)
            lp = logits.ctypes.data_as(_lib.f32p)
        check(lib().glmx_engine_decode(self.h, st, out, lp))
        toks = [[out[i * m + s] for s in range(steps[i])] for i in range(n)]
        return (toks, logits) if want_logits else toks

    def decode_async(self, steps):
        """Enqueue the greedy decode of the last staged batch (see decode), merged with a
        deferred batch's rows if decode_defer() set one aside; collect with decode_collect().
        The next prefill may be staged in between."""
        self._dec_steps = list(steps)
        self._dec_prev = getattr(self, "_def_steps", None)
        self._def_steps = None
        st = (C.c_uint32 * max(1, len(steps)))(*steps)
        check(lib().glmx_engine_decode_async(self.h, st))

    def decode_defer(self, steps):
        """Set the staged batch's decode aside: it runs merged with the next decode_async."""
        self._def_steps = list(steps)
        st = (C.c_uint32 * max(1, len(steps)))(*steps)
        check(lib().glmx_engine_decode_defer(self.h, st))

    def decode_collect(self):
        """Tokens of the collected decode: (tokens of the staged batch, tokens of the merged
        deferred batch or None)."""
        steps, prev = self._dec_steps, self._dec_prev
        m = max(steps + (prev or [])) if (steps or prev) else 0
        out = (C.c_int32 * max(1, len(steps) * m))()
        outp = (C.c_int32 * max(1, len(prev) * m))() if prev else None
        check(lib().glmx_engine_decode_collect(self.h, out, outp))
        cur = [[out[i * m + s] for s in range(steps[i])] for i in range(len(steps))]
        old = [[outp[i * m + s] for s in range(prev[i])] for i in range(len(prev))] if prev else None
        return cur, old

    def io_bytes(self):
        """(host->device, device->host) bytes moved by the engine since creation."""
        out = (C.c_uint64 * 2)()
        check(lib().glmx_engine_io_bytes(self.h, out))
        return int(out[0]), int(out[1])

    def last_timings(self):
        out = (C.c_float * 7)()
        lib().glmx_engine_last_timings(self.h, out)
        keys = ("forward", "attention", "kv_append", "gemm", "elementwise", "h2d", "d2h")
        return dict(zip(keys, list(out)))

    def last_work(self):
        out = (C.c_double * 6)()
        lib().glmx_engine_last_work(self.h, out)
        keys = ("attn_flops", "attn_bytes", "append_bytes", "linear_flops", "computed_tokens",
                "context_tokens")
        return dict(zip(keys, list(out)))
