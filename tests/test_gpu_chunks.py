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
                toks = oracle.tokenize(want)
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
