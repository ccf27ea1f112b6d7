"""CPU checks: the oracle itself (C restatement vs golden + compiled reference), the templates
and tokenizer (a1/a2/a3), the C-ABI library (loads, exports every symbol include/glmx.h
declares, compute entry points refuse to run without a device), and the host graph ingest."""
import ctypes as C
import json
import os
import random
import re

import pytest

import oracle
import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200 import _lib
from paper_2511_01633_b200.templates import TemplateSet

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- the oracle, pinned
def test_port_chain_ids_and_fnv(port, golden):
    toks = [f"t{i}" for i in range(64)]
    assert [str(x) for x in oracle.port_chain_ids(toks)] == golden["chain_ids"]
    assert port.glmo_fnv1a(b"", 0, 14695981039346656037) == 14695981039346656037
    assert port.glmo_fnv1a(b"a", 1, 14695981039346656037) == 0xaf63dc4c8601ec8c


def test_port_prefill_kats(port, golden):
    for kat in golden["prefill_kats"]:
        kv = oracle.PortKv(port, kat["cap"], kat["B"], kat["policy"])
        res = []
        for toks, tiers, sess in kat["ops"]:
            st, rep, ev = kv.prefill(toks, [tuple(t) for t in tiers], sess)
            res.append([st, list(rep), [str(e) for e in ev]])
        assert res == kat["results"]
        assert kv.counters() == kat["counters"]


def test_port_matches_reference_random(ref, port):
    for seed in range(20):
        rnd = random.Random(seed)
        cap, B, pol = rnd.randint(1, 10), rnd.randint(1, 4), rnd.randint(0, 1)
        a, b = oracle.RefKv(ref, cap, B, pol), oracle.PortKv(port, cap, B, pol)
        for _ in range(150):
            p = [f"w{rnd.randint(0, 4)}" for _ in range(rnd.randint(0, 14))]
            t = [(0, len(p), rnd.randint(0, 3))] if p else []
            s = rnd.choice("xyz")
            ra, rb = a.prefill(p, t, s), b.prefill(p, t, s)
            assert ra == rb
            if rnd.random() < 0.1:
                a.set_tier(s, 1, 2)
                b.set_tier(s, 1, 2)
        assert a.resident() == b.resident() and a.counters() == b.counters()


def test_golden_node_info_matches_fixture(golden):
    # SPEC.md:207 / :216 examples, as produced by the reference
    d = {(r[0], r[1], r[2], r[3]): r[4] for r in golden["node_info"]}
    assert d[("n1", 8, 0, False)] == (
        "[Node:n1 {brand:X, price:10, title:alpha widget, type:item}]\n"
        "[neighbours:(n3 {brand:Y, price:11, title:gamma widget, type:item}),(u1 {name:u, type:user})]")
    assert d[("n3", 0, 0, False)].endswith("[neighbours:]")


# ---------------------------------------------------------------- a1/a2/a3 host logic
def test_templates_match_reference(ref):
    t = TemplateSet()
    cases = [("classification", ("What is the price of x?",)),
             ("reasoning", ("Q?", "[Node:n1 {a:b}]\n[neighbours:]\n")),
             ("reasoning", ("Q?", "")),
             ("action", ("vertex chunks for: a; b",)),
             ("action_repair", ("t", "print(x)", "boom")),
             ("baseline_thought", ("Q?", "Thought: x\n")),
             ("baseline_action", ("Q?", ""))]
    for name, args in cases:
        mine = getattr(t, "render_" + name)(*args)
        a = list(args) + [""] * (3 - len(args))
        assert [tuple(x) for x in oracle.ref_render(name, *a)] == mine, name


def test_tokenizer_matches_reference_spans(ref):
    """glmx_tokenize (and the Python restatement) against the reference's glm::tokenize itself
    (tokenizer.hpp:14-25, std::isspace in the C locale), incl. bytes >= 0x80 and NBSP."""
    rnd = random.Random(0)
    alphabet = "ab \t\n\r\x0b\x0cxyz{}[](),:é\xa0"
    for _ in range(300):
        s = "".join(rnd.choice(alphabet) for _ in range(rnd.randint(0, 40)))
        want = oracle.ref_tokenize(s)
        assert glmx.tokenize(s) == want
        assert oracle.tokenize(s) == want


def test_malformed_attribute_rejected_like_reference(ref):
    path = os.path.join(ROOT, "tests", "golden", "attrs_nested.jsonl")
    with pytest.raises(ValueError) as ref_err:
        oracle.RefGraph(path=path)
    with pytest.raises(glmx.GlmxError) as err:
        glmx.PropertyGraph.load(path, device=-1)
    assert str(ref_err.value) in str(err.value)  # same line, same message


# ---------------------------------------------------------------- the C-ABI boundary
def declared_functions():
    with open(os.path.join(ROOT, "include", "glmx.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(glmx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = glmx.lib()
    decl = declared_functions()
    assert len(decl) >= 45
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.EXPORTED)
    assert glmx.lib().glmx_version().decode().startswith("glmx")


def test_compute_entry_points_refuse_without_device(tmp_path):
    """No CPU fallback: compute on a bookkeeping-only handle fails loudly."""
    L = glmx.lib()
    cfg = glmx.TINY.to_c()
    h = C.c_void_p()
    assert L.glmx_model_create(C.byref(cfg), -1, C.byref(h)) == _lib.ERR_NO_DEVICE
    g = glmx.PropertyGraph.load(os.path.join(GOLDEN, "tiny.jsonl"), device=-1)
    r = glmx.Retriever(g, chunk_k=8)
    with pytest.raises(glmx.GlmxError) as e:
        r.node_info_rendered("n1")
    assert e.value.code == _lib.ERR_NO_DEVICE
    kv = glmx.KvCacheState(8, 16)
    m = C.c_void_p()
    ecfg = _lib.EngineConfig(1, 16, 1, 64)
    assert L.glmx_engine_create(m, kv.h, C.byref(ecfg), C.byref(h)) == _lib.ERR_NO_DEVICE


def test_host_graph_ingest_matches_reference(ref, tmp_path):
    g = glmx.PropertyGraph.load(os.path.join(GOLDEN, "tiny.jsonl"), device=-1)
    rg = oracle.RefGraph(path=os.path.join(GOLDEN, "tiny.jsonl"))
    assert [g.node_id(i) for i in range(g.node_count())] == rg.node_ids()
    assert g.total_degree(g.node_index("n3")) == 2 and g.node_index("zz") == -1
    s = glmx.PropertyGraph.synth_powerlaw(3000, 6, seed=11, device=-1)
    p = str(tmp_path / "s.jsonl")
    s.save(p)
    rs = oracle.RefGraph(path=p)
    assert rs.node_ids() == [s.node_id(i) for i in range(s.node_count())]
    s2 = glmx.PropertyGraph.load(p, device=-1)
    assert s2.edge_count() == s.edge_count() == 3000 * 6
    # malformed records are rejected like graph_store.cpp:38-106
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"kind":"node","id":"a","type":"t"}\n{"kind":"edge","src":"a","dst":"b","etype":"x"}\n')
    with pytest.raises(glmx.GlmxError) as e:
        glmx.PropertyGraph.load(str(bad), device=-1)
    assert e.value.code == _lib.ERR_MALFORMED
    dup = tmp_path / "dup.jsonl"
    dup.write_text('{"kind":"node","id":"a","type":"t"}\n{"kind":"node","id":"a","type":"t"}\n')
    with pytest.raises(glmx.GlmxError):
        glmx.PropertyGraph.load(str(dup), device=-1)
