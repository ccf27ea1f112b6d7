"""Configuration C1 end to end on the GPU: the tiny fixture graph, the tiny random-init decoder and
the Fig. 6 ScriptedProvider trace (sessions s1, s2, d1) driven through the
reference's Orchestrator state machine (paper_2511_01633_b200/scripted.py) over the engine.

Checked against the reference itself (tests/golden/golden.json, recorded from oracle/_ref's
orchestrator by make_golden.py): the PromptSegments of every prefill, per-call records (actor,
tokens in / out, cached, computed), answers, the final KV snapshot; and against the CPU fp32
decoder oracle: the logits of every prefill (max-abs 2e-2 + rel 1e-2) and the greedy reply tokens
(bit-exact except at fp32 near-ties)."""
import json
import os

import numpy as np
import pytest

import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200 import scripted as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ATOL, RTOL = 2e-2, 1e-2


def test_output_parsers_and_snippet_subset():
    assert S.parse_classification(" Yes, directly") is True
    assert S.parse_classification("no\n") is False
    with pytest.raises(S.UnexpectedAgentOutput):
        S.parse_classification("maybe")
    assert S.parse_reasoning("x\nMissing: a\nFinish: b\n") == ("finish", "b")
    assert S.parse_reasoning("Missing:  a b \n") == ("missing", "a b")
    assert S.parse_action("pre\n```python\nprint(1)\n```\n") == "print(1)\n"
    assert S.snippet_statements('print(NodeInfo(RetrieveNode("a \\"q\\"")))\n') == [
        ("info", ['a "q"'], None)]
    assert S.snippet_statements('print(NodeFeature([RetrieveNode("a"), RetrieveNode("b")], '
                                '"price"))') == [("feature", ["a", "b"], "price")]
    with pytest.raises(NotImplementedError):
        S.snippet_statements("x = 1")
    tr = S.export_trace([("s", "reasoning", "A"), ("s", "action", "B"), ("s", "reasoning", "C")])
    assert [(t["agent"], t["step"]) for t in tr] == [("reasoning", 0), ("action", 0),
                                                       ("reasoning", 1)]


def run_c1(want_logits=True):
    cfg = glmx.TINY
    g = glmx.PropertyGraph.load(os.path.join(GOLDEN, "tiny.jsonl"), device=0)
    model = glmx.Model(cfg, device=0)
    kv = glmx.KvCacheState(4096, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                           n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, headroom_pages=64)
    eng = glmx.Engine(model, kv, max_requests=8, max_batch_tokens=2048, max_decode=32,
                      max_context=1024)
    ret = glmx.Retriever(g, chunk_k=8, vocab=cfg.vocab)
    wl = S.ScriptedWorkload(eng, ret, glmx.NodeIndex(g),
                            S.load_trace(os.path.join(GOLDEN, "fig6_trace.jsonl")),
                            S.load_questions(os.path.join(GOLDEN, "fig6_questions.jsonl")),
                            lanes=8, want_logits=want_logits)
    calls = wl.run()
    return model, kv, wl, calls


@pytest.mark.gpu
def test_c1_fig6_end_to_end(golden):
    from oracle.decoder import Decoder, token_ids

    f = golden["fig6"]
    model, kv, wl, calls = run_c1()
    # the reference's prefill sequence: same segments, same order
    ref_prefills = [t for t in f["trace"] if t["op"] == "prefill"]
    assert len(calls) == len(ref_prefills) == 10
    for c, t in zip(calls, ref_prefills):
        assert c.session.sid == t["session"]
        assert [(tier, text) for tier, text in c.segments] == [
            (tier, text) for text, tier in t["segments"] if text]
        assert c.tokens == t["tokens"]
        assert (c.report.cached_tokens, c.report.computed_tokens, c.report.tail_tokens) == (
            t["cached"], t["computed"], t["tail"])
    # per-session records / answers (the V records are retrieval timing only)
    for s, ref_s in zip(wl.sessions, f["sessions"]):
        assert s.sid == ref_s["id"] and s.answer == ref_s["answer"]
        assert [r.row() for r in s.records] == [r[:5] for r in ref_s["records"] if r[0] != "V"]
        assert [r.outcome for r in s.records][0] == ref_s["records"][0][6]
    assert kv.snapshot() == f["kv"]
    # tensor math against the CPU fp32 decoder: logits of every prefill, greedy reply tokens
    dec = Decoder(model.cfg, model.export_all())
    n_tie = 0
    for c in calls:
        ids = token_ids(c.tokens, model.cfg.vocab)
        ref_logits, _ = dec.forward(ids)
        err = np.abs(c.logits - ref_logits)
        assert np.all(err <= ATOL + RTOL * np.abs(ref_logits)), (c.session.sid, err.max())
        n_tie += dec.check_greedy(ids, [c.first_token] + c.decoded)
    assert sum(len(c.decoded) for c in calls) == sum(
        r[2] - 1 for s in f["sessions"] for r in s["records"] if r[0] != "V")
    print("C1: near-tie exemptions", n_tie)
