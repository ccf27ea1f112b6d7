"""K1 vertex-chunk assembly on the GPU vs the reference Retriever::node_info_rendered
(retriever.cpp:74-129) compiled from /root/reference (oracle/_ref): byte-exact chunks and
token streams (tokenizer.hpp:14-25), for every node of the fixture and sampled nodes (hubs
included) of a seeded power-law graph, across k, weight modes and directedness."""
import os
import random

import pytest

import oracle
import paper_2511_01633_b200 as glmx
from oracle.decoder import fnv1a

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_fixture_chunks_match_reference(ref):
    path = os.path.join(GOLDEN, "tiny.jsonl")
    g = glmx.PropertyGraph.load(path, device=0)
    rg = oracle.RefGraph(path=path)
    ids = rg.node_ids()
    assert [g.node_id(i) for i in range(g.node_count())] == ids
    for k in (0, 1, 2, 8, -3):
        for wm in (0, 1):
            for directed in (False, True):
                r = glmx.Retriever(g, chunk_k=k, weight_mode=wm, directed=directed, vocab=32000)
                for nid in ids:
                    assert r.node_info_rendered(nid) == rg.node_info_rendered(nid, k, wm, directed)
    r = glmx.Retriever(g, chunk_k=8)
    with pytest.raises(glmx.RetrievalError):
        r.node_info_rendered("nope")
    # SPEC.md:207 / SURVEY Appendix C golden
    assert r.node_info_rendered("n1") == (
        "[Node:n1 {brand:X, price:10, title:alpha widget, type:item}]\n"
        "[neighbours:(n3 {brand:Y, price:11, title:gamma widget, type:item}),(u1 {name:u, type:user})]")


def test_attribute_rendering_matches_reference(ref):
    """attr.hpp:19-48 + retriever.cpp:34-41 (SURVEY trap A11): doubles in shortest round-trip form
    (1e+21, 0.1, -0, 1e-07, 5e-324, DBL_MAX, integers beyond int64 as doubles, 100.0 -> 100),
    uint64 values wrapped to int64, bools, lists (empty, mixed), an attribute literally named
    `type` (two type pairs, sorted by value), non-ASCII / escaped / whitespace-bearing strings,
    multi-edges and a self-loop: chunk bytes, token spans and token ids per node, every k /
    weight mode / direction, against the compiled reference."""
    path = os.path.join(GOLDEN, "attrs.jsonl")
    g = glmx.PropertyGraph.load(path, device=0)
    rg = oracle.RefGraph(path=path)
    ids = rg.node_ids()
    assert [g.node_id(i) for i in range(g.node_count())] == ids
    V = 32000
    for k in (0, 1, 2, 8):
        for wm in (0, 1):
            for directed in (False, True):
                r = glmx.Retriever(g, chunk_k=k, weight_mode=wm, directed=directed, vocab=V)
                batch = r.chunk_build(list(range(len(ids))))
                for i, nid in enumerate(ids):
                    want = rg.node_info_rendered(nid, k, wm, directed)
                    assert r.node_info_rendered(nid) == want
                    assert batch.texts[i] == want
                    raw = want.encode()
                    toks = oracle.ref_tokenize(raw)
                    assert [raw[b:e] for b, e in batch.token_spans[i]] == toks
                    assert batch.token_ids[i] == [fnv1a(t) % V for t in toks]


def test_batched_chunks_and_tokens_match_reference(ref, tmp_path):
    g = glmx.PropertyGraph.synth_powerlaw(20000, 8, seed=3, device=0)
    path = str(tmp_path / "g.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    n = g.node_count()
    rnd = random.Random(0)
    nodes = list(range(12)) + [rnd.randrange(n) for _ in range(300)] + [n - 1]
    V = 128256
    for k in (0, 1, 8, 16, 64):
        for wm, directed in ((0, False), (1, False), (0, True)):
            r = glmx.Retriever(g, chunk_k=k, weight_mode=wm, directed=directed, vocab=V)
            batch = r.chunk_build(nodes)
            for i, v in enumerate(nodes):
                want = rg.node_info_rendered(g.node_id(v), k, wm, directed)
                assert batch.texts[i] == want, (k, wm, directed, v)
                toks = oracle.ref_tokenize(want)  # the reference's glm::tokenize
                got = [batch.texts[i].encode()[b:e].decode() for b, e in batch.token_spans[i]]
                assert got == toks
                assert batch.token_ids[i] == [fnv1a(t.encode()) % V for t in toks]


def test_hub_rows_stream_through_window(ref, tmp_path):
    # node 0 of the power-law graph has in-degree >> the 1024-key sort window
    g = glmx.PropertyGraph.synth_powerlaw(50000, 8, seed=5, device=0)
    assert g.total_degree(0) > 2048
    path = str(tmp_path / "g.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    for k in (1, 16, 64, 300):
        r = glmx.Retriever(g, chunk_k=k)
        for v in (0, 1, 2):
            assert r.node_info_rendered(g.node_id(v)) == rg.node_info_rendered(g.node_id(v), k)


def test_whitespace_edge_cases_tokens_match_reference(ref, tmp_path):
    """Attribute values with tabs, newlines, runs of spaces, leading/trailing blanks, no blanks at
    all and non-ASCII bytes: chunk text and whitespace tokens (spans + fnv1a ids) fused across
    entry boundaries exactly as the reference tokenizer splits them; includes chunks larger than
    the 4 KB shared-memory staging buffer (built and tokenised in place in global memory)."""
    import json

    rnd = random.Random(11)
    tab, nl, cr = chr(9), chr(10), chr(13)
    vals = ["plain", "two words", "  lead", "trail  ", "tab" + tab + "sep", "new" + nl + "line",
            "cr" + cr + "lf" + nl, "multi   space", "", " ", "caf" + chr(233), "x" * 40, "abc",
            "end,", "(paren)", "}{"]
    lines = []
    n_nodes = 400
    for i in range(n_nodes):
        attrs = {f"k{j}": rnd.choice(vals) for j in range(rnd.randrange(0, 4))}
        if i % 7 == 0:
            attrs["blob"] = " ".join(rnd.choice(vals) for _ in range(60))  # long entries
        lines.append(json.dumps({"kind": "node", "id": f"v{i:04d}",
                                 "type": rnd.choice(["a", "b c"]), "attrs": attrs}))
    for i in range(n_nodes):
        for _ in range(rnd.randrange(1, 6)):
            lines.append(json.dumps({"kind": "edge", "src": f"v{i:04d}",
                                     "dst": f"v{rnd.randrange(10):04d}", "etype": "e"}))
    path = str(tmp_path / "ws.jsonl")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    g = glmx.PropertyGraph.load(path, device=0)
    rg = oracle.RefGraph(path=path)
    V = 128256
    nodes = list(range(g.node_count()))
    for k in (3, 16, 64, 200):
        r = glmx.Retriever(g, chunk_k=k, vocab=V)
        batch = r.chunk_build(nodes)
        big = 0
        for i, v in enumerate(nodes):
            want = rg.node_info_rendered(g.node_id(v), k)
            assert batch.texts[i] == want, (k, v)
            big += len(want.encode()) > 4096
            toks = oracle.ref_tokenize(want)  # the reference's glm::tokenize
            raw = batch.texts[i].encode()
            got = [raw[b:e].decode() for b, e in batch.token_spans[i]]
            assert got == toks, (k, v)
            assert batch.token_ids[i] == [fnv1a(t.encode()) % V for t in toks]
        if k == 200:
            assert big > 0  # the unstaged path ran


def test_irregular_entries_take_byte_tokenizer(ref, tmp_path):
    """K1 has two tokenizers: the table-driven one for chunks whose entries are all regular
    (first and last byte non-space, >= 2 tokens; DevGraph::ent_head) and the byte-level one for
    the rest.  Node ids that start with whitespace make their entries irregular: batches mixing
    such chunks with regular ones (neighbour lists of both kinds, k across a 32-piece round and
    a 4 KB staging buffer) give the reference's bytes and tokens from both paths."""
    import json

    rnd = random.Random(5)
    ids = [f"r{i:03d}" for i in range(150)] + [" s1", "\tt2", "  u3", " " * 3 + "w4", "\nx5"]
    lines = [json.dumps({"kind": "node", "id": nid, "type": rnd.choice(["item", "user"]),
                         "attrs": {"title": " ".join(f"w{rnd.randrange(99)}"
                                                     for _ in range(rnd.randrange(1, 30)))}})
             for nid in ids]
    for nid in ids:
        for _ in range(rnd.randrange(1, 40)):
            lines.append(json.dumps({"kind": "edge", "src": nid, "dst": rnd.choice(ids),
                                     "etype": rnd.choice(["e", "f"])}))
    path = str(tmp_path / "irr.jsonl")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    g = glmx.PropertyGraph.load(path, device=0)
    rg = oracle.RefGraph(path=path)
    V = 128256
    nodes = list(range(g.node_count()))
    for k in (0, 1, 5, 31, 32, 33, 80):
        r = glmx.Retriever(g, chunk_k=k, vocab=V)
        batch = r.chunk_build(nodes)
        for i, v in enumerate(nodes):
            want = rg.node_info_rendered(g.node_id(v), k)
            assert batch.texts[i] == want, (k, v)
            toks = oracle.ref_tokenize(want)
            raw = want.encode()
            assert [raw[b:e] for b, e in batch.token_spans[i]] == [t.encode() for t in toks], (k, v)
            assert batch.token_ids[i] == [fnv1a(t.encode()) % V for t in toks]
        # vocab 0: no ids, same spans
        r0 = glmx.Retriever(g, chunk_k=k, vocab=0)
        b0 = r0.chunk_build(nodes)
        assert b0.token_spans == batch.token_spans and b0.texts == batch.texts


def test_fill_call_after_other_batch_is_rebuilt(ref, tmp_path):
    """glmx_chunk_build's fill call reuses the size query's result only for the same node list and
    configuration: a size query for one batch followed by a fill call for another (or for the same
    nodes under another k / vocab) returns the second batch's chunks."""
    import ctypes as C

    from paper_2511_01633_b200._lib import check, lib

    g = glmx.PropertyGraph.synth_powerlaw(3000, 6, seed=2, device=0)
    path = str(tmp_path / "g.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    a, b = [5, 17, 300], [9, 9, 2000, 41]
    r16 = glmx.Retriever(g, chunk_k=16, vocab=32000)
    r4 = glmx.Retriever(g, chunk_k=4, vocab=32000)

    def fill(r, nodes):
        n = len(nodes)
        arr = (C.c_int32 * n)(*nodes)
        tb, tt = C.c_uint64(), C.c_uint64()
        out = C.create_string_buffer(1 << 16)
        boff = (C.c_uint64 * (n + 1))()
        check(lib().glmx_chunk_build(g.h, C.byref(r.cfg), arr, n, out, 1 << 16, boff, None, None,
                                     None, 0, None, C.byref(tb), C.byref(tt)))
        raw = out.raw
        return [raw[boff[i]:boff[i + 1]].decode() for i in range(n)]

    for size_r, size_nodes, fill_r, fill_nodes, k in ((r16, a, r16, b, 16), (r16, b, r4, b, 4)):
        n = len(size_nodes)
        arr = (C.c_int32 * n)(*size_nodes)
        tb, tt = C.c_uint64(), C.c_uint64()
        check(lib().glmx_chunk_build(g.h, C.byref(size_r.cfg), arr, n, None, 0, None, None, None,
                                     None, 0, None, C.byref(tb), C.byref(tt)))
        got = fill(fill_r, fill_nodes)
        assert got == [rg.node_info_rendered(g.node_id(v), k) for v in fill_nodes]


def test_large_batch_grows_buffers_on_device_overflow(ref, tmp_path):
    """A batch whose size bound exceeds the preallocated outputs (12000 chunks at k=64) takes the
    device overflow path: the render sees the capacities, raises the flag, and the host grows the
    buffers and renders again; every chunk (sampled against the reference) and the token stream
    come out as from small batches."""
    g = glmx.PropertyGraph.synth_powerlaw(20000, 8, seed=9, device=0)
    path = str(tmp_path / "g.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    rnd = random.Random(3)
    nodes = [rnd.randrange(g.node_count()) for _ in range(12000)]
    V = 128256
    r = glmx.Retriever(g, chunk_k=64, vocab=V)
    big = r.chunk_build(nodes)
    small = r.chunk_build(nodes[:50])
    assert big.texts[:50] == small.texts and big.token_ids[:50] == small.token_ids
    for i in rnd.sample(range(len(nodes)), 40):
        want = rg.node_info_rendered(g.node_id(nodes[i]), 64)
        assert big.texts[i] == want
        raw = want.encode()
        assert [raw[b:e] for b, e in big.token_spans[i]] == oracle.ref_tokenize(raw)
