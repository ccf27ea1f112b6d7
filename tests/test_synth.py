"""The pure-Python workload definitions both bench arms share (paper_2511_01633_b200/synth.py):
the graph JSONL is byte-identical to the C++ generator + serializer the GPU arm loads, the
question stream is the one GraphCoTWorkload drives, and the reference's own PropertyGraph::load
reads the file back with the same node order."""
import pytest

import oracle
import paper_2511_01633_b200 as glmx
from paper_2511_01633_b200 import synth


@pytest.mark.parametrize("n,e,seed", [(2000, 8, 0), (1003, 3, 7), (12, 2, 5)])
def test_graph_jsonl_identical_to_cpp_generator(tmp_path, n, e, seed):
    g = glmx.PropertyGraph.synth_powerlaw(n, e, seed=seed, device=-1)
    a, b = str(tmp_path / "a.jsonl"), str(tmp_path / "b.jsonl")
    g.save(a)
    synth.powerlaw_graph_jsonl(n, e, seed, b)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_reference_loads_the_synthetic_graph(ref, tmp_path):
    path = synth.powerlaw_graph_jsonl(500, 4, 3, str(tmp_path / "g.jsonl"))
    assert oracle.RefGraph(path=path).node_ids() == [synth.node_id(i) for i in range(500)]


def test_question_stream_is_prefix_stable_and_repeats():
    a = synth.graph_cot_questions(100000, 400, 0, repeat_frac=0.22)
    b = synth.graph_cot_questions(100000, 1000, 0, repeat_frac=0.22)
    assert b[:400] == a
    uniq = len({q for _, _, q in b}) / len(b)
    assert 0.74 <= uniq <= 0.82  # ~22% repeats, like the reference's generate_workload
    assert synth.graph_cot_questions(1000, 50, 1, question_pool=10)[:20] == \
        synth.graph_cot_questions(1000, 20, 1, question_pool=10)
    tr = synth.scripted_replies(a[:2])
    assert [t["agent"] for t in tr if t["session"] == a[0][0]][:3] == [
        "classification", "reasoning", "action"]
