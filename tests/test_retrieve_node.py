"""RetrieveNode (retriever.cpp:49-66, index.cpp:41-56, embedder.cpp:19-36).

CPU: the host embedding equals the reference's bit for bit (texts with and without trigrams,
multibyte UTF-8, several dims).  GPU (K5): the device nearest scan returns exactly the
reference's VectorIndex::nearest(text, 1) — including ties, which break by ascending id — and the
retrieval LRU reproduces the reference's hit/miss/probe counts."""
import random
import struct

import pytest

import oracle
import paper_2511_01633_b200 as glmx

TEXTS = ["alpha widget", "", "ab", "abc", "umber lattice v0000012", "user v0000019", "zzzz",
         "héllo wörld", "  spaced   text  ", "Which item is linked from all of: a; b?"]


def bits(xs):
    return [struct.unpack("<I", struct.pack("<f", x))[0] for x in xs]


@pytest.mark.parametrize("dim", [64, 13, 128])
def test_embedding_bit_exact(ref, dim):
    rnd = random.Random(dim)
    texts = TEXTS + ["".join(chr(rnd.randrange(32, 127)) for _ in range(rnd.randrange(0, 60)))
                     for _ in range(50)]
    for t in texts:
        assert bits(glmx.embed(t, dim)) == bits(oracle.ref_embed(t, dim)), t


@pytest.mark.gpu
def test_retrieve_matches_reference_nearest(ref, tmp_path):
    g = glmx.PropertyGraph.synth_powerlaw(6000, 8, seed=11, device=0)
    path = str(tmp_path / "g.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    idx = glmx.NodeIndex(g)
    assert len(idx) == g.node_count()  # every synthetic node has a title or a name
    rnd = random.Random(1)
    titles = []
    for _ in range(40):
        v = rnd.randrange(g.node_count())
        info = g.node_id(v)
        titles.append(info)
    queries = TEXTS + titles + ["widget", "cobalt gasket", "user", "v00001", "ochre brazier v00"]
    got, hits = idx.retrieve_nodes(queries)
    assert not any(hits[:len(set(queries))])  # all first lookups miss
    for q, v in zip(queries, got):
        want = rg.nearest(q, 1)[0]
        assert g.node_id(v) == want, (q, g.node_id(v), want)


@pytest.mark.gpu
def test_retrieval_lru_counts(ref):
    g = glmx.PropertyGraph.synth_powerlaw(2000, 4, seed=3, device=0)
    idx = glmx.NodeIndex(g, cache_capacity=3)
    seq = ["a b c", "d e f", "a b c", "g h i", "j k l", "d e f", "a b c", "a b c"]
    # reference LruCache(3): miss, miss, hit, miss, miss (evicts d e f), miss, miss (a b c was
    # evicted by the put of d e f), hit
    ids, hits = idx.retrieve_nodes(seq[:4])
    ids2, hits2 = idx.retrieve_nodes(seq[4:])
    assert hits + hits2 == [False, False, True, False, False, False, False, True]
    assert idx.stats() == (2, 6, 6)
    assert ids[0] == ids[2] == ids2[2] == ids2[3]


@pytest.mark.gpu
@pytest.mark.parametrize("nodes,n,ratio", [(500, 200, 0.5), (1200, 400, 0.25), (300, 64, 0.0)])
def test_generate_workload_matches_reference(ref, tmp_path, nodes, n, ratio):
    """Scalable generate_workload: identical JSONL to the reference's on its own synthetic
    graph (synth_graph(seed 7), the C3 workload source), pools validated by one GPU scan."""
    from paper_2511_01633_b200.retrieve import generate_workload

    rg = oracle.RefGraph(synth=(7, nodes))
    path = str(tmp_path / "synth.jsonl")
    rg.save(path)
    g = glmx.PropertyGraph.load(path, device=0)
    want = rg.generate_workload(7, n, ratio)
    got, ms = generate_workload(g, 7, n, ratio)
    assert got == want
    assert ms > 0


@pytest.mark.gpu
def test_generate_workload_errors_match(ref, tmp_path):
    from paper_2511_01633_b200.retrieve import generate_workload

    g = glmx.PropertyGraph.synth_powerlaw(800, 4, seed=2, device=0)
    path = str(tmp_path / "p.jsonl")
    g.save(path)
    rg = oracle.RefGraph(path=path)
    for ratio in (0.0, 0.5):
        try:
            want = rg.generate_workload(3, 100, ratio)
        except LookupError as e:
            with pytest.raises(glmx.GlmxError) as ei:
                generate_workload(g, 3, 100, ratio)
            assert str(e) in str(ei.value)
            continue
        got, _ = generate_workload(g, 3, 100, ratio)
        assert got == want
