"""Python mirror of the reference's KvCacheState (cache.hpp:56-99) over the C-ABI.

Same names, argument meaning and error behaviour: ``prefill(tokens, tiers, session)`` returns a
PrefillReport, raises CacheExhausted with partial state left, GlmxError(ERR_GLM) for a bad
TierMap, ConfigError for block size 0.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

from . import _lib
from ._lib import check, lib

TIER_I, TIER_II, TIER_III, TIER_IV = 0, 1, 2, 3
PRIORITY, PLAIN_LRU = 0, 1


@dataclass
class PrefillReport:
    cached_tokens: int = 0
    computed_tokens: int = 0
    tail_tokens: int = 0
    evicted: list = field(default_factory=list)
    block_table: list = field(default_factory=list)

    def total_computed(self):
        return self.computed_tokens + self.tail_tokens


def pack_tokens(tokens):
    bs = [t.encode() if isinstance(t, str) else bytes(t) for t in tokens]
    blob = b"".join(bs)
    offs = (C.c_uint64 * (len(bs) + 1))()
    o = 0
    for i, b in enumerate(bs):
        offs[i] = o
        o += len(b)
    offs[len(bs)] = o
    return blob, offs


def pack_tiers(tiers):
    arr = (_lib.TierRange * max(1, len(tiers)))()
    for i, (b, e, t) in enumerate(tiers):
        arr[i].begin, arr[i].end, arr[i].tier = b, e, t
    return arr


def chain_ids(tokens, block_tokens=16):
    """KvCacheState::chain_ids (cache.cpp:31-40)."""
    blob, offs = pack_tokens(tokens)
    out = (C.c_uint64 * (len(tokens) // max(1, block_tokens) + 1))()
    n = lib().glmx_kv_chain_ids(blob, offs, len(tokens), block_tokens, out)
    return [out[i] for i in range(n)]


def count_tokens(text: str) -> int:
    """count_tokens (tokenizer.hpp:36-46): std::isspace-delimited tokens, through the C-ABI."""
    b = text.encode()
    return int(lib().glmx_tokenize(b, len(b), None, None, 0))


def tokenize(text: str):
    """tokenizer.hpp:14-25 through the C-ABI."""
    b = text.encode()
    n = lib().glmx_tokenize(b, len(b), None, None, 0)
    beg, end = (C.c_uint64 * max(1, n))(), (C.c_uint64 * max(1, n))()
    lib().glmx_tokenize(b, len(b), beg, end, n)
    return [b[beg[i]:end[i]].decode() for i in range(n)]


class KvCacheState:
    def __init__(self, capacity_blocks, block_tokens=16, policy=PRIORITY, device=-1,
                 n_layers=0, n_kv_heads=0, head_dim=0, headroom_pages=0):
        cfg = _lib.KvConfig(capacity_blocks, block_tokens, policy, device, n_layers, n_kv_heads,
                            head_dim, headroom_pages)
        h = C.c_void_p()
        check(lib().glmx_kv_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.block_tokens = block_tokens
        self.capacity_blocks = capacity_blocks
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().glmx_kv_destroy(self.h)
            self.h = None

    __del__ = _lib.safe_del

    def prefill(self, tokens, tiers, session) -> PrefillReport:
        blob, offs = pack_tokens(tokens)
        tarr = pack_tiers(tiers)
        rep = _lib.PrefillReportC()
        nb = len(tokens) // self.block_tokens
        bt = (C.c_int32 * max(1, nb))()
        cap = nb + 8
        ev = (C.c_uint64 * cap)()
        check(lib().glmx_kv_prefill(self.h, blob, offs, len(tokens), tarr, len(tiers),
                                    session.encode(), C.byref(rep), bt, nb, ev, cap))
        evicted = self._evicted(rep.n_evicted, ev, cap)
        return PrefillReport(rep.cached_tokens, rep.computed_tokens, rep.tail_tokens, evicted,
                             [bt[i] for i in range(rep.n_blocks)])

    def prefill_segments(self, segments, session) -> PrefillReport:
        """Orchestrator::kv_prefill (orchestrator.cpp:81-97): [(tier, text), ...]."""
        texts = [t.encode() for _, t in segments]
        n = len(segments)
        arr = (C.c_char_p * max(1, n))(*texts)
        lens = (C.c_uint64 * max(1, n))(*[len(t) for t in texts])
        tiers = (C.c_int32 * max(1, n))(*[t for t, _ in segments])
        rep = _lib.PrefillReportC()
        nb = sum(len(t) for t in texts) // self.block_tokens + 1
        bt = (C.c_int32 * nb)()
        cap = nb + 8
        ev = (C.c_uint64 * cap)()
        check(lib().glmx_kv_prefill_segments(self.h, n, arr, lens, tiers, session.encode(),
                                             C.byref(rep), bt, nb, ev, cap))
        return PrefillReport(rep.cached_tokens, rep.computed_tokens, rep.tail_tokens,
                             self._evicted(rep.n_evicted, ev, cap),
                             [bt[i] for i in range(rep.n_blocks)])

    def _evicted(self, n, ev, cap):
        if n <= cap:
            return [ev[i] for i in range(n)]
        full = (C.c_uint64 * n)()
        lib().glmx_kv_last_evicted(self.h, full, n)
        return list(full)

    def evict(self, n):
        out = (C.c_uint64 * max(1, n))()
        got = C.c_uint64()
        check(lib().glmx_kv_evict(self.h, n, out, n, C.byref(got)))
        return [out[i] for i in range(got.value)]

    def set_tier(self, session, from_tier, to_tier):
        check(lib().glmx_kv_set_tier(self.h, session.encode(), from_tier, to_tier))

    def force_insert(self, block_id, tier, last_used, session):
        check(lib().glmx_kv_force_insert(self.h, block_id, tier, last_used, session.encode()))

    def counters(self):
        out = (C.c_int64 * 6)()
        lib().glmx_kv_counters(self.h, out)
        return {"hits": out[0], "misses": out[1], "evictions_by_tier": list(out[2:6])}

    def hit_rate(self):
        c = self.counters()
        t = c["hits"] + c["misses"]
        return 0.0 if t == 0 else c["hits"] / t

    def resident_blocks(self):
        return lib().glmx_kv_resident(self.h, None, None, None, None, 0)

    def resident_snapshot(self):
        n = self.resident_blocks()
        ids, tiers = (C.c_uint64 * max(1, n))(), (C.c_int32 * max(1, n))()
        lu, pages = (C.c_uint64 * max(1, n))(), (C.c_int32 * max(1, n))()
        lib().glmx_kv_resident(self.h, ids, tiers, lu, pages, n)
        return [(ids[i], tiers[i], lu[i], pages[i]) for i in range(n)]

    def is_resident(self, block_id):
        return self.block_session(block_id) is not None

    def block_session(self, block_id):
        buf = C.create_string_buffer(4096)
        n = lib().glmx_kv_block_session(self.h, block_id, buf, 4096)
        return None if n < 0 else buf.raw[:n].decode()

    def snapshot_json(self):
        buf = C.create_string_buffer(4096)
        n = lib().glmx_kv_snapshot_json(self.h, buf, 4096)
        return buf.raw[:n].decode()

    def snapshot(self):
        return json.loads(self.snapshot_json())

    # ---- cross-GPU prefix hits ----------------------------------------------
    def resident_ids_pages(self):
        """(block ids uint64[n], pages int32[n]) of the residents — this rank's directory entry."""
        import numpy as np

        n = self.resident_blocks()
        ids = np.zeros(max(1, n), dtype=np.uint64)
        pages = np.zeros(max(1, n), dtype=np.int32)
        lib().glmx_kv_resident(self.h, ids.ctypes.data_as(_lib.u64p), None, None,
                               pages.ctypes.data_as(_lib.i32p), n)
        return ids[:n], pages[:n]

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(lib().glmx_kv_ipc_handle(self.h, buf))
        return bytes(buf)

    def attach_peer(self, peer: int, handle: bytes):
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        check(lib().glmx_kv_attach_peer(self.h, peer, buf))

    def attach_peer_local(self, peer: int, other: "KvCacheState"):
        check(lib().glmx_kv_attach_peer_local(self.h, peer, other.h))

    def set_peer_directory(self, ids, peers, pages):
        import numpy as np

        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        peers = np.ascontiguousarray(peers, dtype=np.int32)
        pages = np.ascontiguousarray(pages, dtype=np.int32)
        check(lib().glmx_kv_set_peer_directory(self.h, len(ids), ids.ctypes.data_as(_lib.u64p),
                                               peers.ctypes.data_as(_lib.i32p),
                                               pages.ctypes.data_as(_lib.i32p)))

    def set_epoch_mode(self, on=True):
        check(lib().glmx_kv_set_epoch_mode(self.h, int(on)))

    def release_deferred(self):
        check(lib().glmx_kv_release_deferred(self.h))

    def defer_mark(self) -> int:
        """Number of pages deferred so far (pipelined epochs release with a lag)."""
        return lib().glmx_kv_defer_mark(self.h)

    def release_deferred_before(self, mark: int):
        check(lib().glmx_kv_release_deferred_before(self.h, mark))

    def peer_hits(self):
        return lib().glmx_kv_peer_hits(self.h)

    def pool_pages(self):
        return lib().glmx_kv_pool_pages(self.h)

    def free_pages(self):
        return lib().glmx_kv_free_pages(self.h)
