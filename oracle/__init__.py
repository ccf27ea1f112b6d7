"""TEST INFRASTRUCTURE ONLY — the checkers for the GLM prefill hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this package, and only as the checker or the timed CPU baseline, never as the thing
measured or shipped.

* ``ref()``  -> ctypes over ``oracle/_ref/libglmref.so``: the reference C++ itself
  (/root/reference/proj/src, unmodified) plus ``ref_shim.cpp``.
* ``port()`` -> ctypes over ``oracle/_build/libglm_oracle.so``: the plain-C restatement
  (``glm_oracle.c``) of cache.cpp / fnv.hpp / retriever.cpp.
* ``decoder`` -> numpy fp32 Llama-style decoder (builder-authored: the reference has no tensor
  math, SPEC.md:22 / :547, so the attention / logits / greedy-id oracle is *parity unpinned* by
  the reference and pinned only to the reference's token/block layout).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libglmref.so")
PORT_SO = os.path.join(HERE, "_build", "libglm_oracle.so")
REFERENCE_ROOT = "/root/reference/proj"

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


def build(ref: bool = True) -> None:
    """Build the C restatement, and the reference when its sources are present (this container)."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref and os.path.isdir(REFERENCE_ROOT):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "-j8"], check=True)
        # the compiled drop-in proof (reference run_bench over integration/'s KvCacheState)
        subprocess.run(["make", "-s", "-C", HERE, "dropin", "-j8"], check=True)


def pack_tokens(tokens):
    """list[str|bytes] -> (bytes blob, uint64[n+1] offsets) as ctypes objects."""
    bs = [t.encode() if isinstance(t, str) else bytes(t) for t in tokens]
    blob = b"".join(bs)
    offs = (C.c_uint64 * (len(bs) + 1))()
    o = 0
    for i, b in enumerate(bs):
        offs[i] = o
        o += len(b)
    offs[len(bs)] = o
    return C.create_string_buffer(blob, len(blob) + 1), offs


def pack_tiers(tiers):
    arr = (C.c_uint64 * (3 * max(1, len(tiers))))()
    for i, (b, e, t) in enumerate(tiers):
        arr[3 * i], arr[3 * i + 1], arr[3 * i + 2] = b, e, t
    return arr


class _KvBase:
    """Common Python face over the two CPU KV checkers (reference and C port)."""

    def prefill(self, tokens, tiers, session):
        blob, offs = pack_tokens(tokens)
        tarr = pack_tiers(tiers)
        rep = (C.c_uint64 * 3)()
        cap = len(tokens) + 64 + 4 * max(0, self._resident_hint())
        ev = (C.c_uint64 * cap)()
        nev = C.c_uint64()
        st = self._prefill(blob, offs, len(tokens), tarr, len(tiers), session.encode(), rep, ev,
                           cap, C.byref(nev))
        return st, (rep[0], rep[1], rep[2]), [ev[i] for i in range(min(nev.value, cap))]

    def _resident_hint(self):
        return 0


class RefKv(_KvBase):
    def __init__(self, lib, cap, block_tokens=16, policy=0):
        self.L = lib
        self.h = lib.ref_kv_create(cap, block_tokens, policy)
        if not self.h:
            raise ValueError(lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_kv_destroy(self.h)
            self.h = None

    def _prefill(self, *a):
        return self.L.ref_kv_prefill(self.h, *a)

    def _resident_hint(self):
        return self.resident_count()

    def evict(self, n):
        out = (C.c_uint64 * max(1, n))()
        nout = C.c_uint64()
        st = self.L.ref_kv_evict(self.h, n, out, n, C.byref(nout))
        return st, [out[i] for i in range(nout.value if st == 0 else 0)]

    def set_tier(self, session, frm, to):
        self.L.ref_kv_set_tier(self.h, session.encode(), frm, to)

    def force_insert(self, bid, tier, last_used, session):
        self.L.ref_kv_force_insert(self.h, bid, tier, last_used, session.encode())

    def counters(self):
        out = (C.c_int64 * 6)()
        self.L.ref_kv_counters(self.h, out)
        return list(out)

    def resident_count(self):
        return self.L.ref_kv_resident(self.h, None, None, None, None, 0)

    def resident(self):
        n = self.resident_count()
        ids, tiers = (C.c_uint64 * max(1, n))(), (C.c_int32 * max(1, n))()
        lu, par = (C.c_uint64 * max(1, n))(), (C.c_uint64 * max(1, n))()
        self.L.ref_kv_resident(self.h, ids, tiers, lu, par, n)
        return [(ids[i], tiers[i], lu[i]) for i in range(n)]

    def block_session(self, bid):
        buf = C.create_string_buffer(4096)
        n = self.L.ref_kv_block_session(self.h, bid, buf, 4096)
        return None if n < 0 else buf.raw[:n].decode()

    def snapshot_json(self):
        buf = C.create_string_buffer(1 << 16)
        n = self.L.ref_kv_snapshot_json(self.h, buf, 1 << 16)
        return json.loads(buf.raw[:n].decode())


class PortKv(_KvBase):
    def __init__(self, lib, cap, block_tokens=16, policy=0):
        self.L = lib
        self.h = lib.glmo_kv_create(cap, block_tokens, policy)
        if not self.h:
            raise ValueError("block size must be positive")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.glmo_kv_destroy(self.h)
            self.h = None

    def _prefill(self, *a):
        return self.L.glmo_kv_prefill(self.h, *a)

    def _resident_hint(self):
        return self.resident_count()

    def evict(self, n):
        out = (C.c_uint64 * max(1, n))()
        nout = C.c_size_t()
        st = self.L.glmo_kv_evict(self.h, n, out, n, C.byref(nout))
        return st, [out[i] for i in range(nout.value if st == 0 else 0)]

    def set_tier(self, session, frm, to):
        self.L.glmo_kv_set_tier(self.h, session.encode(), frm, to)

    def force_insert(self, bid, tier, last_used, session):
        self.L.glmo_kv_force_insert(self.h, bid, tier, last_used, session.encode())

    def counters(self):
        out = (C.c_int64 * 6)()
        self.L.glmo_kv_counters(self.h, out)
        return list(out)

    def resident_count(self):
        return self.L.glmo_kv_resident(self.h, None, None, None, 0)

    def resident(self):
        n = self.resident_count()
        ids, tiers, lu = (C.c_uint64 * max(1, n))(), (C.c_int32 * max(1, n))(), (C.c_uint64 * max(1, n))()
        self.L.glmo_kv_resident(self.h, ids, tiers, lu, n)
        return [(ids[i], tiers[i], lu[i]) for i in range(n)]


_ref = None
_port = None


def ref():
    """The compiled reference (oracle/_ref). Raises FileNotFoundError when not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_kv_create.restype = C.c_void_p
        L.ref_kv_create.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.ref_kv_destroy.argtypes = [C.c_void_p]
        L.ref_kv_prefill.argtypes = [C.c_void_p, C.c_char_p, u64p, C.c_uint64, u64p, C.c_uint64,
                                     C.c_char_p, u64p, u64p, C.c_uint64, u64p]
        L.ref_kv_evict.argtypes = [C.c_void_p, C.c_uint64, u64p, C.c_uint64, u64p]
        L.ref_kv_set_tier.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
        L.ref_kv_force_insert.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_char_p]
        L.ref_kv_counters.argtypes = [C.c_void_p, i64p]
        L.ref_kv_resident.restype = C.c_uint64
        L.ref_kv_resident.argtypes = [C.c_void_p, u64p, i32p, u64p, u64p, C.c_uint64]
        L.ref_kv_block_session.restype = C.c_int64
        L.ref_kv_block_session.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_kv_snapshot_json.restype = C.c_int64
        L.ref_kv_snapshot_json.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        L.ref_chain_ids.restype = C.c_uint64
        L.ref_chain_ids.argtypes = [C.c_char_p, u64p, C.c_uint64, C.c_uint64, u64p]
        L.ref_graph_load.restype = C.c_void_p
        L.ref_graph_load.argtypes = [C.c_char_p]
        L.ref_synth_graph.restype = C.c_void_p
        L.ref_synth_graph.argtypes = [C.c_uint64, C.c_int]
        L.ref_graph_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_node_count.restype = C.c_uint64
        L.ref_graph_node_count.argtypes = [C.c_void_p]
        L.ref_graph_node_id.restype = C.c_int64
        L.ref_graph_node_id.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_node_info_rendered.restype = C.c_int64
        L.ref_node_info_rendered.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                             C.c_char_p, C.c_uint64]
        L.ref_retrieve_node.restype = C.c_int64
        L.ref_retrieve_node.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_uint64]
        L.ref_embed.restype = C.c_int64
        L.ref_embed.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_float), C.c_uint64]
        L.ref_generate_workload.restype = C.c_int64
        L.ref_generate_workload.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_double, C.c_char_p,
                                            C.c_uint64]
        L.ref_nearest.restype = C.c_int64
        L.ref_nearest.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_char_p, C.c_uint64]
        L.ref_tokenize.restype = C.c_uint64
        L.ref_tokenize.argtypes = [C.c_char_p, C.c_uint64, u64p, u64p, C.c_uint64]
        L.ref_render.restype = C.c_int64
        L.ref_render.argtypes = [C.c_char_p] * 4 + [C.c_char_p, C.c_uint64]
        L.ref_trace_len.restype = C.c_uint64
        L.ref_trace_line.restype = C.c_int64
        L.ref_trace_line.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_run_bench.restype = C.c_int64
        L.ref_run_bench.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_double, C.c_int,
                                    C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_uint64]
        L.ref_run_scripted.restype = C.c_int64
        L.ref_run_scripted.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_uint64,
                                       C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_uint64]
        L.ref_scripted_open.restype = C.c_void_p
        L.ref_scripted_open.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_uint64,
                                        C.c_int, C.c_int]
        L.ref_scripted_rotation.restype = C.c_int64
        L.ref_scripted_rotation.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        L.ref_scripted_snapshot.restype = C.c_int64
        L.ref_scripted_snapshot.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        L.ref_scripted_close.argtypes = [C.c_void_p]
        _ref = L
    return _ref


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise FileNotFoundError(PORT_SO)
        L = C.CDLL(PORT_SO)
        L.glmo_fnv1a.restype = C.c_uint64
        L.glmo_fnv1a.argtypes = [C.c_char_p, C.c_size_t, C.c_uint64]
        L.glmo_fnv1a_u64.restype = C.c_uint64
        L.glmo_fnv1a_u64.argtypes = [C.c_uint64, C.c_uint64]
        L.glmo_chain_ids.restype = C.c_size_t
        L.glmo_chain_ids.argtypes = [C.c_char_p, u64p, C.c_size_t, C.c_size_t, u64p]
        L.glmo_kv_create.restype = C.c_void_p
        L.glmo_kv_create.argtypes = [C.c_size_t, C.c_size_t, C.c_int]
        L.glmo_kv_destroy.argtypes = [C.c_void_p]
        L.glmo_kv_prefill.argtypes = [C.c_void_p, C.c_char_p, u64p, C.c_size_t, u64p, C.c_size_t,
                                      C.c_char_p, u64p, u64p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.glmo_kv_evict.argtypes = [C.c_void_p, C.c_size_t, u64p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.glmo_kv_set_tier.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
        L.glmo_kv_force_insert.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_char_p]
        L.glmo_kv_counters.argtypes = [C.c_void_p, i64p]
        L.glmo_kv_resident.restype = C.c_size_t
        L.glmo_kv_resident.argtypes = [C.c_void_p, u64p, i32p, u64p, C.c_size_t]
        L.glmo_node_info_rendered.restype = C.c_int64
        _port = L
    return _port


def ref_embed(text, dim=64):
    """The reference's embed(text, dim) (embedder.cpp:19-36) as a list of floats (padded)."""
    L = ref()
    out = (C.c_float * 1024)()
    n = L.ref_embed(text.encode(), dim, out, 1024)
    return [out[i] for i in range(n)]


def ref_chain_ids(tokens, block_tokens=16):
    L = ref()
    blob, offs = pack_tokens(tokens)
    out = (C.c_uint64 * (len(tokens) // block_tokens + 1))()
    n = L.ref_chain_ids(blob, offs, len(tokens), block_tokens, out)
    return [out[i] for i in range(n)]


def port_chain_ids(tokens, block_tokens=16):
    L = port()
    blob, offs = pack_tokens(tokens)
    out = (C.c_uint64 * (len(tokens) // block_tokens + 1))()
    n = L.glmo_chain_ids(blob, offs, len(tokens), block_tokens, out)
    return [out[i] for i in range(n)]


class RefGraph:
    def __init__(self, path=None, synth=None):
        L = ref()
        self.L = L
        if path is not None:
            self.h = L.ref_graph_load(path.encode())
        else:
            self.h = L.ref_synth_graph(synth[0], synth[1])
        if not self.h:
            raise ValueError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_graph_free(self.h)
            self.h = None

    def save(self, path):
        assert self.L.ref_graph_save(self.h, path.encode()) == 0

    def node_ids(self):
        n = self.L.ref_graph_node_count(self.h)
        buf = C.create_string_buffer(4096)
        out = []
        for i in range(n):
            m = self.L.ref_graph_node_id(self.h, i, buf, 4096)
            out.append(buf.raw[:m].decode())
        return out

    def node_info_rendered(self, node_id, k=8, weight_mode=0, directed=False):
        cap = 1 << 20
        buf = C.create_string_buffer(cap)
        n = self.L.ref_node_info_rendered(self.h, node_id.encode(), k, weight_mode, int(directed),
                                          buf, cap)
        if n < 0:
            raise LookupError(self.L.ref_last_error().decode())
        if n > cap:
            buf = C.create_string_buffer(n)
            n = self.L.ref_node_info_rendered(self.h, node_id.encode(), k, weight_mode,
                                              int(directed), buf, n)
        return buf.raw[:n].decode()

    def nearest(self, text, k):
        """VectorIndex::nearest(text, k) ids (index built once per call, default Config)."""
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        n = self.L.ref_nearest(self.h, text.encode(), k, buf, cap)
        if n < 0:
            raise LookupError(self.L.ref_last_error().decode())
        return buf.raw[:n].decode().split("\n") if n else []

    def generate_workload(self, seed, n, ratio):
        """generate_workload(...).serialize_jsonl() of the reference (workload.cpp:158-255)."""
        cap = 1 << 24
        buf = C.create_string_buffer(cap)
        m = self.L.ref_generate_workload(self.h, seed, n, ratio, buf, cap)
        if m < 0:
            raise LookupError(self.L.ref_last_error().decode())
        return buf.raw[:m].decode()

    def retrieve_node(self, text):
        buf = C.create_string_buffer(4096)
        n = self.L.ref_retrieve_node(self.h, text.encode(), buf, 4096)
        if n < 0:
            raise LookupError(self.L.ref_last_error().decode())
        return buf.raw[:n].decode()

    def run_bench(self, seed=7, n=200, ratio=0.5, concurrency=8, cap=4096, policy=0, glm=True,
                  record=False):
        L = self.L
        L.ref_trace_clear()
        buf = C.create_string_buffer(1 << 20)
        m = L.ref_run_bench(self.h, seed, n, ratio, concurrency, cap, policy, int(glm),
                            int(record), buf, 1 << 20)
        if m < 0:
            raise RuntimeError(L.ref_last_error().decode())
        return json.loads(buf.raw[:m].decode()), (trace_lines() if record else None)

    def run_scripted(self, trace_path, questions, concurrency=8, cap=4096, policy=0, chunk_k=8,
                     record=False):
        L = self.L
        L.ref_trace_clear()
        qs = "\n".join(json.dumps(q) for q in questions)
        cap_out = 1 << 24
        buf = C.create_string_buffer(cap_out)
        m = L.ref_run_scripted(self.h, trace_path.encode(), qs.encode(), concurrency, cap, policy,
                               chunk_k, int(record), buf, cap_out)
        if m < 0:
            raise RuntimeError(L.ref_last_error().decode())
        return json.loads(buf.raw[:m].decode()), (trace_lines() if record else None)


class RefScriptedRun:
    """The reference's Orchestrator + ScriptedProvider + KvCacheState + Retriever (oracle/_ref)
    over a graph, driven one round-robin rotation at a time (bench.cpp:71-83)."""

    def __init__(self, graph, trace_path, questions, lanes=8, cap=4096, policy=0, chunk_k=8):
        L = ref()
        self.L, self.graph = L, graph
        qs = "\n".join(json.dumps(q) for q in questions)
        self.h = L.ref_scripted_open(graph.h, trace_path.encode(), qs.encode(), lanes, cap, policy,
                                     chunk_k)
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())
        self.done = False

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_scripted_close(self.h)
            self.h = None

    def rotation(self):
        """Runs one rotation; returns its calls [(session, actor, cached, computed+tail)]."""
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        m = self.L.ref_scripted_rotation(self.h, buf, cap)
        if m < 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        out = json.loads(buf.raw[:m].decode())
        self.done = out["done"]
        return [tuple(c) for c in out["calls"]]

    def snapshot(self):
        buf = C.create_string_buffer(4096)
        n = self.L.ref_scripted_snapshot(self.h, buf, 4096)
        return json.loads(buf.raw[:n].decode())


def trace_lines():
    L = ref()
    n = L.ref_trace_len()
    out = []
    cap = 1 << 22
    buf = C.create_string_buffer(cap)
    for i in range(n):
        m = L.ref_trace_line(i, buf, cap)
        out.append(json.loads(buf.raw[:m].decode()))
    return out


def ref_render(name, a0="", a1="", a2=""):
    L = ref()
    cap = 1 << 20
    buf = C.create_string_buffer(cap)
    n = L.ref_render(name.encode(), a0.encode(), a1.encode(), a2.encode(), buf, cap)
    if n < 0:
        raise ValueError(L.ref_last_error().decode())
    return [(t, txt) for t, txt in json.loads(buf.raw[:n].decode())]


def ref_tokenize(text):
    """The reference's own glm::tokenize (tokenizer.hpp:14-25) through oracle/_ref: the tokens of
    `text` (str or bytes) as the same type."""
    L = ref()
    raw = text.encode() if isinstance(text, str) else bytes(text)
    cap = len(raw) // 2 + 2
    b, e = (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
    n = L.ref_tokenize(raw, len(raw), b, e, cap)
    assert n <= cap
    toks = [raw[b[i]:e[i]] for i in range(n)]
    return [t.decode() for t in toks] if isinstance(text, str) else toks


def tokenize(text: str):
    """tokenizer.hpp:14-25 restated: split on std::isspace (C locale: ' \\t\\n\\v\\f\\r')."""
    out = []
    i, n = 0, len(text)
    ws = " \t\n\v\f\r"
    while i < n:
        while i < n and text[i] in ws:
            i += 1
        s = i
        while i < n and text[i] not in ws:
            i += 1
        if i > s:
            out.append(text[s:i])
    return out


def kv_prefill_inputs(segments):
    """orchestrator.cpp:81-97 restated: per-segment tokenisation, same-tier range merge."""
    tokens, tiers = [], []
    for tier, text in segments:
        part = tokenize(text)
        if not part:
            continue
        b = len(tokens)
        tokens += part
        if tiers and tiers[-1][2] == tier:
            tiers[-1][1] = len(tokens)
        else:
            tiers.append([b, len(tokens), tier])
    return tokens, [tuple(t) for t in tiers]
