"""glmx — B200-native prefill over a paged KV pool with vertex-chunk prefix reuse.

Drop-in for the hot path of the GLM reference (arXiv 2511.01633, /root/reference/proj): the
vertex-chunk builder, prefix-cache lookup/insert, four-tier priority eviction and the
prefill/decode step, as a C-ABI library (include/glmx.h, libglmx.so) with hand-written sm_100a
kernels.  This package is the thin ctypes face used by tests and bench.py.
"""
from ._lib import (CacheExhausted, ConfigError, GlmxError, RetrievalError, lib)  # noqa: F401
from .kvcache import (PLAIN_LRU, PRIORITY, TIER_I, TIER_II, TIER_III, TIER_IV,  # noqa: F401
                      KvCacheState, PrefillReport, chain_ids, tokenize)
from .model import LLAMA3_8B, TINY, Engine, Model, ModelConfig, Request  # noqa: F401
from .retrieve import (BY_EDGE_TYPE, TOTAL_DEGREE, NodeIndex, PropertyGraph, Retriever,  # noqa: F401
                       embed)
