"""a17 / C3 parity: the Graph-CoT workload driven over the engine (pipelined rotations, one prefill
batch per rotation, in-batch finish) against the reference's OWN Orchestrator + ScriptedProvider
+ KvCacheState + Retriever (oracle/_ref) fed the same graph JSONL, questions and replies
(paper_2511_01633_b200/synth.py), rotation by rotation: identical calls in identical order with
identical cached / computed tokens, and the same final cache snapshot -- under eviction pressure
with four-tier priority eviction, and with plain LRU."""
import os

import pytest

import oracle
import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200 import synth
from paper_2511_01633_b200.workload import GraphCoTWorkload

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cap,policy", [(4096, 0), (64, 0), (48, 1)],
                         ids=["roomy", "priority_pressure", "lru_pressure"])
def test_workload_matches_reference_orchestrator(ref, tmp_path, cap, policy):
    n_nodes, seed, lanes, n_q = 3000, 4, 16, 48
    gpath = synth.powerlaw_graph_jsonl(n_nodes, 6, seed, str(tmp_path / "g.jsonl"))
    g = glmx.PropertyGraph.load(gpath, device=0)
    cfg = glmx.TINY
    model = glmx.Model(cfg, device=0)
    kv = glmx.KvCacheState(cap, 16, policy, device=0, n_layers=cfg.n_layers,
                           n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, headroom_pages=2048)
    eng = glmx.Engine(model, kv, max_requests=lanes, max_batch_tokens=lanes * 1024, max_decode=4,
                      max_context=4096)
    wl = GraphCoTWorkload(eng, glmx.Retriever(g, chunk_k=8, vocab=cfg.vocab), n_queries=n_q,
                          lanes=lanes, seed=5, question_pool=20, node_index=glmx.NodeIndex(g))
    sessions = [(s.sid, s.sources, s.question) for s in wl.sessions]
    assert sessions == synth.graph_cot_questions(n_nodes, n_q, 5, question_pool=20)
    ours = []
    while not wl.done():
        ours.extend(wl.rotations(1))
    tpath = synth.write_jsonl(synth.scripted_replies(sessions), str(tmp_path / "trace.jsonl"))
    run = oracle.RefScriptedRun(oracle.RefGraph(path=gpath), tpath,
                                [{"id": sid, "text": q} for sid, _, q in sessions], lanes, cap,
                                policy, 8)
    theirs = []
    while not run.done:
        theirs.append(run.rotation())
    assert len(ours) == len(theirs)
    for i, (a, b) in enumerate(zip(ours, theirs)):
        got = [(c.session.sid, {"classification": "C", "reasoning": "R", "action": "A"}[c.agent],
                rep.cached_tokens, rep.computed_tokens + rep.tail_tokens)
               for c, rep in zip(a.calls_made, a.reports)]
        assert got == b, i
    assert kv.snapshot() == run.snapshot()
    if cap < 4096:
        assert sum(kv.counters()["evictions_by_tier"]) > 0
    model.close()
