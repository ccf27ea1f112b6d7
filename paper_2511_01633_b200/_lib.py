"""ctypes binding of include/glmx.h (libglmx.so, built in-tree).

The product path has no fallback: if the shared library is missing or fails to load, importing
any engine class raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GLMX_LIB selects a diagnostics build (libglmx_trace.so); the default is the product library
LIB_PATH = os.environ.get("GLMX_LIB") or os.path.join(HERE, "libglmx.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
f32p = C.POINTER(C.c_float)

OK = 0
ERR_GLM = 1
ERR_CACHE_EXHAUSTED = 2
ERR_CONFIG = 3
ERR_RETRIEVAL = 4
ERR_CUDA = 5
ERR_ARG = 6
ERR_NO_DEVICE = 7
ERR_MALFORMED = 8
ERR_POOL = 9


class KvConfig(C.Structure):
    _fields_ = [("capacity_blocks", C.c_uint64), ("block_tokens", C.c_uint32),
                ("policy", C.c_int32), ("device", C.c_int32), ("n_layers", C.c_uint32),
                ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32),
                ("headroom_pages", C.c_uint64)]


class TierRange(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64), ("tier", C.c_int32),
                ("reserved", C.c_int32)]


class PrefillReportC(C.Structure):
    _fields_ = [("cached_tokens", C.c_uint64), ("computed_tokens", C.c_uint64),
                ("tail_tokens", C.c_uint64), ("n_evicted", C.c_uint64), ("n_blocks", C.c_uint64)]


class ChunkConfig(C.Structure):
    _fields_ = [("k", C.c_int32), ("weight_mode", C.c_int32), ("directed", C.c_int32),
                ("vocab", C.c_uint32)]


class ModelConfigC(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("d_model", C.c_uint32), ("n_heads", C.c_uint32),
                ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32), ("d_ff", C.c_uint32),
                ("vocab", C.c_uint32), ("rope_theta", C.c_float), ("norm_eps", C.c_float),
                ("init_std", C.c_float), ("seed", C.c_uint64)]


class EngineConfig(C.Structure):
    _fields_ = [("max_requests", C.c_uint32), ("max_batch_tokens", C.c_uint32),
                ("max_decode", C.c_uint32), ("max_context", C.c_uint32)]


class RequestC(C.Structure):
    _fields_ = [("tok_bytes", C.c_char_p), ("tok_offsets", u64p), ("n_tok", C.c_uint64),
                ("tiers", C.POINTER(TierRange)), ("n_tiers", C.c_uint64),
                ("session", C.c_char_p), ("finish", C.c_int32)]


class SegmentRequestC(C.Structure):
    _fields_ = [("seg_text", C.POINTER(C.c_char_p)), ("seg_len", u64p), ("seg_tier", i32p),
                ("n_seg", C.c_uint64), ("session", C.c_char_p), ("finish", C.c_int32)]


_SIGS = {
    "glmx_last_error": (C.c_char_p, []),
    "glmx_version": (C.c_char_p, []),
    "glmx_device_count": (C.c_int, []),
    "glmx_kv_create": (C.c_int, [C.POINTER(KvConfig), C.POINTER(C.c_void_p)]),
    "glmx_kv_destroy": (None, [C.c_void_p]),
    "glmx_kv_prefill": (C.c_int, [C.c_void_p, C.c_char_p, u64p, C.c_uint64, C.POINTER(TierRange),
                                  C.c_uint64, C.c_char_p, C.POINTER(PrefillReportC), i32p,
                                  C.c_uint64, u64p, C.c_uint64]),
    "glmx_kv_prefill_segments": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_char_p), u64p,
                                           i32p, C.c_char_p, C.POINTER(PrefillReportC), i32p,
                                           C.c_uint64, u64p, C.c_uint64]),
    "glmx_kv_last_evicted": (C.c_uint64, [C.c_void_p, u64p, C.c_uint64]),
    "glmx_kv_evict": (C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_uint64, u64p]),
    "glmx_kv_set_tier": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32]),
    "glmx_kv_force_insert": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.c_uint64, C.c_char_p]),
    "glmx_kv_counters": (C.c_int, [C.c_void_p, i64p]),
    "glmx_kv_resident": (C.c_uint64, [C.c_void_p, u64p, i32p, u64p, i32p, C.c_uint64]),
    "glmx_kv_block": (C.c_int32, [C.c_void_p, C.c_uint64, i32p, u64p, u64p, i32p]),
    "glmx_kv_block_session": (C.c_int64, [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64]),
    "glmx_kv_snapshot_json": (C.c_int64, [C.c_void_p, C.c_char_p, C.c_uint64]),
    "glmx_kv_chain_ids": (C.c_uint64, [C.c_char_p, u64p, C.c_uint64, C.c_uint32, u64p]),
    "glmx_kv_release_deferred": (C.c_int, [C.c_void_p]),
    "glmx_kv_defer_mark": (C.c_uint64, [C.c_void_p]),
    "glmx_kv_release_deferred_before": (C.c_int, [C.c_void_p, C.c_uint64]),
    "glmx_kv_pool_pages": (C.c_uint64, [C.c_void_p]),
    "glmx_kv_free_pages": (C.c_uint64, [C.c_void_p]),
    "glmx_kv_pool_ptr": (C.c_void_p, [C.c_void_p]),
    "glmx_kv_page_bytes": (C.c_uint64, [C.c_void_p]),
    "glmx_kv_ipc_handle": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "glmx_kv_attach_peer": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint8)]),
    "glmx_kv_attach_peer_local": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "glmx_kv_set_peer_directory": (C.c_int, [C.c_void_p, C.c_uint64, u64p, i32p, i32p]),
    "glmx_kv_set_epoch_mode": (C.c_int, [C.c_void_p, C.c_int32]),
    "glmx_kv_peer_hits": (C.c_int64, [C.c_void_p]),
    "glmx_tokenize": (C.c_uint64, [C.c_char_p, C.c_uint64, u64p, u64p, C.c_uint64]),
    "glmx_token_id": (C.c_int32, [C.c_char_p, C.c_uint64, C.c_uint32]),
    "glmx_graph_load_jsonl": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "glmx_graph_synth_powerlaw": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int32,
                                            C.POINTER(C.c_void_p)]),
    "glmx_graph_save_jsonl": (C.c_int, [C.c_void_p, C.c_char_p]),
    "glmx_graph_destroy": (None, [C.c_void_p]),
    "glmx_graph_node_count": (C.c_uint64, [C.c_void_p]),
    "glmx_graph_edge_count": (C.c_uint64, [C.c_void_p]),
    "glmx_graph_node_index": (C.c_int64, [C.c_void_p, C.c_char_p]),
    "glmx_graph_node_id": (C.c_int64, [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64]),
    "glmx_graph_degree": (C.c_int64, [C.c_void_p, C.c_uint64]),
    "glmx_graph_io_bytes": (C.c_int, [C.c_void_p, u64p]),
    "glmx_graph_node_attr": (C.c_int64, [C.c_void_p, C.c_uint64, C.c_char_p, C.c_char_p,
                                         C.c_uint64, i32p]),
    "glmx_chunk_build": (C.c_int, [C.c_void_p, C.POINTER(ChunkConfig), i32p, C.c_uint64,
                                   C.c_char_p, C.c_uint64, u64p, i32p, u64p, u64p, C.c_uint64,
                                   u64p, u64p, u64p]),
    "glmx_node_info_rendered": (C.c_int64, [C.c_void_p, C.POINTER(ChunkConfig), C.c_char_p,
                                            C.c_char_p, C.c_uint64]),
    "glmx_chunk_last_kernel_ms": (C.c_float, [C.c_void_p]),
    "glmx_model_create": (C.c_int, [C.POINTER(ModelConfigC), C.c_int32, C.POINTER(C.c_void_p)]),
    "glmx_model_destroy": (None, [C.c_void_p]),
    "glmx_model_export_weight": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32,
                                           C.POINTER(C.c_uint16), C.c_uint64]),
    "glmx_model_tune_gemms": (C.c_int, [C.c_void_p, C.c_int32, i32p]),
    "glmx_engine_create": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(EngineConfig),
                                     C.POINTER(C.c_void_p)]),
    "glmx_engine_destroy": (None, [C.c_void_p]),
    "glmx_engine_prefill": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(RequestC),
                                      C.POINTER(PrefillReportC), i32p, f32p]),
    "glmx_engine_prefill_segments": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(SegmentRequestC),
                                               C.POINTER(PrefillReportC), i32p, f32p]),
    "glmx_engine_prefill_segments_async": (C.c_int, [C.c_void_p, C.c_uint64,
                                                     C.POINTER(SegmentRequestC),
                                                     C.POINTER(PrefillReportC)]),
    "glmx_engine_wait": (C.c_int, [C.c_void_p, i32p, C.c_uint64]),
    "glmx_engine_in_flight": (C.c_int32, [C.c_void_p]),
    "glmx_engine_decode": (C.c_int, [C.c_void_p, u32p, i32p, f32p]),
    "glmx_engine_decode_async": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "glmx_engine_decode_collect": (C.c_int, [C.c_void_p, i32p, i32p]),
    "glmx_engine_decode_defer": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "glmx_engine_io_bytes": (C.c_int, [C.c_void_p, u64p]),
    "glmx_engine_last_timings": (C.c_int, [C.c_void_p, f32p]),
    "glmx_engine_last_work": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "glmx_engine_set_profiling": (None, [C.c_void_p, C.c_int32]),
    "glmx_engine_set_reuse": (None, [C.c_void_p, C.c_int32]),
    "glmx_pool_copy": (C.c_int, [C.c_void_p, C.c_void_p, i32p, i32p, C.c_uint64, C.c_void_p]),
    "glmx_pool_last_copy_ms": (C.c_float, [C.c_void_p]),
    "glmx_rope_kv_append_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                          C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_void_p,
                                          C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                          C.c_int32, C.c_void_p, f32p]),
    "glmx_attn_trace_read": (C.c_int32, [i64p, C.c_int32]),
    "glmx_kv_gather_run": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint32, i32p, C.c_uint64,
                                     C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, f32p]),
    "glmx_attn_schedule": (C.c_int, [i32p, C.c_int32, C.c_int32, i32p, i32p, C.c_int32,
                                     C.c_int32, i32p, i32p, i32p, i32p, i64p]),
    "glmx_index_build": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64]),
    "glmx_index_size": (C.c_uint64, [C.c_void_p]),
    "glmx_workload_generate": (C.c_int64, [C.c_void_p, C.c_uint64, C.c_int32, C.c_double,
                                           C.c_char_p, C.c_uint64, f32p]),
    "glmx_retrieve_nodes": (C.c_int, [C.c_void_p, C.c_char_p, u64p, C.c_uint64, i32p,
                                      C.POINTER(C.c_uint8)]),
    "glmx_retriever_stats": (None, [C.c_void_p, i64p]),
    "glmx_retrieve_last_kernel_ms": (C.c_float, [C.c_void_p]),
    "glmx_embed_text": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int32, f32p]),
    "glmx_attention_run": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32,
                                     C.c_int32, C.c_int32, C.c_void_p, C.c_uint64, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint64, i32p, i32p, i32p, i32p,
                                     C.c_int32, C.c_int32, C.c_void_p, f32p]),
}

EXPORTED = sorted(_SIGS)

_lib = None


def lib():
    """Load libglmx.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def safe_del(self):
    """__del__ for handle owners: close(), ignoring failures at interpreter shutdown (module
    globals such as the loaded library may already be torn down)."""
    try:
        self.close()
    except Exception:  # noqa: BLE001
        pass


class GlmxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class CacheExhausted(GlmxError):
    """KvCacheState's CacheExhausted (error.hpp:110-113)."""


class RetrievalError(GlmxError):
    """RetrievalError (error.hpp:75-80)."""


class ConfigError(GlmxError):
    pass


def check(st):
    if st != OK:
        msg = lib().glmx_last_error().decode(errors="replace")
        cls = {ERR_CACHE_EXHAUSTED: CacheExhausted, ERR_RETRIEVAL: RetrievalError,
               ERR_CONFIG: ConfigError}.get(st, GlmxError)
        raise cls(st, msg)
    return st
