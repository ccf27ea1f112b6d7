"""Python mirror of PropertyGraph (graph_store.hpp:27-75) + Retriever::node_info_rendered
(retriever.cpp:123-129), with the batched vertex-chunk kernel K1 behind glmx_chunk_build."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from ._lib import check, lib

TOTAL_DEGREE, BY_EDGE_TYPE = 0, 1


@dataclass
class ChunkBatch:
    texts: list          # rendered chunk per request (str)
    token_ids: list      # per request list[int] (empty when vocab == 0)
    token_spans: list    # per request list[(begin, end)] byte spans within the chunk
    kernel_ms: float
    nodes: list = None   # node index per chunk (set by the workload driver)


class PropertyGraph:
    def __init__(self, handle):
        self.h = handle

    @classmethod
    def load(cls, path, device=0):
        h = C.c_void_p()
        check(lib().glmx_graph_load_jsonl(path.encode(), device, C.byref(h)))
        return cls(h)

    @classmethod
    def synth_powerlaw(cls, n_nodes, edges_per_node=8, seed=0, device=0):
        h = C.c_void_p()
        check(lib().glmx_graph_synth_powerlaw(n_nodes, edges_per_node, seed, device, C.byref(h)))
        return cls(h)

    def save(self, path):
        check(lib().glmx_graph_save_jsonl(self.h, path.encode()))

    def close(self):
        if getattr(self, "h", None):
            lib().glmx_graph_destroy(self.h)
            self.h = None

    __del__ = _lib.safe_del

    def node_count(self):
        return lib().glmx_graph_node_count(self.h)

    def edge_count(self):
        return lib().glmx_graph_edge_count(self.h)

    def node_index(self, node_id):
        return lib().glmx_graph_node_index(self.h, node_id.encode())

    def node_id(self, idx):
        buf = C.create_string_buffer(4096)
        n = lib().glmx_graph_node_id(self.h, idx, buf, 4096)
        return None if n < 0 else buf.raw[:n].decode()

    def node_attr(self, idx, key):
        """(rendered value, kind) of node idx's attribute `key` (kinds: 0 string, 1 int,
        2 double, 3 bool, 4 list), or None when absent."""
        buf = C.create_string_buffer(4096)
        kind = C.c_int32()
        n = lib().glmx_graph_node_attr(self.h, int(idx), key.encode(), buf, 4096, C.byref(kind))
        if n < 0:
            return None
        if n > 4096:
            buf = C.create_string_buffer(n)
            lib().glmx_graph_node_attr(self.h, int(idx), key.encode(), buf, n, C.byref(kind))
        return buf.raw[:n].decode(), kind.value

    def io_bytes(self):
        """(host->device, device->host) bytes of K1 / K5 calls on this graph since load."""
        out = (C.c_uint64 * 2)()
        check(lib().glmx_graph_io_bytes(self.h, out))
        return int(out[0]), int(out[1])

    def total_degree(self, idx):
        return lib().glmx_graph_degree(self.h, idx)


class Retriever:
    """Vertex-chunk side of the reference Retriever (retriever.hpp:26-72)."""

    def __init__(self, graph: PropertyGraph, chunk_k=8, weight_mode=TOTAL_DEGREE, directed=False,
                 vocab=0):
        self.graph = graph
        self.cfg = _lib.ChunkConfig(chunk_k, weight_mode, int(directed), vocab)

    def node_info_rendered(self, node_id: str) -> str:
        cap = 1 << 16
        while True:
            buf = C.create_string_buffer(cap)
            n = lib().glmx_node_info_rendered(self.graph.h, C.byref(self.cfg), node_id.encode(),
                                              buf, cap)
            if n < 0:
                check(-n)
            if n <= cap:
                return buf.raw[:n].decode()
            cap = n

    def chunk_build(self, node_idx) -> ChunkBatch:
        """K1 over a batch of node indices (one chunk per entry, duplicates allowed)."""
        n = len(node_idx)
        nodes = (C.c_int32 * max(1, n))(*node_idx)
        tb, tt = C.c_uint64(), C.c_uint64()
        check(lib().glmx_chunk_build(self.graph.h, C.byref(self.cfg), nodes, n, None, 0, None,
                                     None, None, None, 0, None, C.byref(tb), C.byref(tt)))
        out = C.create_string_buffer(max(1, tb.value))
        boff = (C.c_uint64 * (n + 1))()
        ntok = max(1, tt.value)
        tid = (C.c_int32 * ntok)()
        tbeg, tend = (C.c_uint64 * ntok)(), (C.c_uint64 * ntok)()
        toff = (C.c_uint64 * (n + 1))()
        check(lib().glmx_chunk_build(self.graph.h, C.byref(self.cfg), nodes, n, out, tb.value,
                                     boff, tid, tbeg, tend, ntok, toff, C.byref(tb), C.byref(tt)))
        raw = out.raw
        texts, ids, spans = [], [], []
        for i in range(n):
            texts.append(raw[boff[i]:boff[i + 1]].decode())
            ids.append([tid[j] for j in range(toff[i], toff[i + 1])] if self.cfg.vocab else [])
            spans.append([(tbeg[j], tend[j]) for j in range(toff[i], toff[i + 1])])
        return ChunkBatch(texts, ids, spans, lib().glmx_chunk_last_kernel_ms(self.graph.h))

    def chunk_build_device(self, node_idx):
        """K1 over a batch without copying the outputs back: (total bytes, total tokens, device ms
        of select -> scans -> render+tokenize).  For measurements."""
        n = len(node_idx)
        nodes = (C.c_int32 * max(1, n))(*node_idx)
        tb, tt = C.c_uint64(), C.c_uint64()
        check(lib().glmx_chunk_build(self.graph.h, C.byref(self.cfg), nodes, n, None, 0, None,
                                     None, None, None, 0, None, C.byref(tb), C.byref(tt)))
        return tb.value, tt.value, lib().glmx_chunk_last_kernel_ms(self.graph.h)


def embed(text: str, dim: int = 64):
    """embed(text, dim) of the reference (embedder.cpp:19-36), host C++: list of padded floats."""
    out = (C.c_float * ((dim + 7) // 8 * 8))()
    b = text.encode()
    check(lib().glmx_embed_text(b, len(b), dim, out))
    return list(out)


class NodeIndex:
    """RetrieveNode over the device-resident VectorIndex of a graph (K5 + the retrieval LRU),
    Retriever::retrieve_node_traced semantics (retriever.cpp:49-66)."""

    def __init__(self, graph: PropertyGraph, dim: int = 64, cache_capacity: int = 1024):
        self.graph = graph
        check(lib().glmx_index_build(graph.h, dim, cache_capacity))

    def __len__(self):
        return lib().glmx_index_size(self.graph.h)

    def retrieve_nodes(self, texts):
        """Resolve texts in order -> (node indices, cache-hit flags)."""
        bs = [t.encode() for t in texts]
        offs = [0]
        for b in bs:
            offs.append(offs[-1] + len(b))
        n = len(bs)
        off_arr = (C.c_uint64 * (n + 1))(*offs)
        out = (C.c_int32 * max(1, n))()
        hit = (C.c_uint8 * max(1, n))()
        check(lib().glmx_retrieve_nodes(self.graph.h, b"".join(bs), off_arr, n, out, hit))
        return [out[i] for i in range(n)], [bool(hit[i]) for i in range(n)]

    def retrieve_node(self, text):
        return self.graph.node_id(self.retrieve_nodes([text])[0][0])

    def stats(self):
        """(cache_hits, cache_misses, index_probes)."""
        out = (C.c_int64 * 3)()
        lib().glmx_retriever_stats(self.graph.h, out)
        return tuple(out)

    def last_kernel_ms(self):
        return lib().glmx_retrieve_last_kernel_ms(self.graph.h)


def generate_workload(graph: PropertyGraph, seed: int, n: int, nondet_ratio: float):
    """The reference's generate_workload (workload.cpp:158-255) at scale: returns (JSONL text in
    Workload::serialize_jsonl's format, device ms of the batched K5 validation scan)."""
    ms = C.c_float(0.0)
    m = lib().glmx_workload_generate(graph.h, seed, n, nondet_ratio, None, 0, C.byref(ms))
    if m < 0:
        check(-m)
    buf = C.create_string_buffer(max(1, m))
    lib().glmx_workload_generate(graph.h, seed, n, nondet_ratio, buf, m, C.byref(ms))
    return buf.raw[:m].decode(), ms.value
