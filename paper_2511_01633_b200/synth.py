"""Synthetic inputs of the C2-C5 configurations, in pure Python (no ctypes, no device): the seeded
power-law property graph, the Graph-CoT question stream and its scripted replies.

Both bench arms build their workload from these definitions: the GPU arm (through the package)
and ``bench.py --impl reference``, which loads this file by path -- never the package, so the
reference arm maps no product library -- and feeds the reference's own PropertyGraph::load,
Orchestrator and ScriptedProvider (oracle/_ref) the same graph, questions and replies.

* ``powerlaw_graph_jsonl`` writes exactly the JSONL of ``glmx_graph_synth_powerlaw`` +
  ``glmx_graph_save_jsonl`` (host/graph.cpp synth_powerlaw / serialize_jsonl; pinned by
  tests/test_synth.py): splitmix64 draws, out-edge targets floor(n * u^3) (hub degree
  ~ n^(2/3)), ids zero-padded so byte order == index order.
* ``graph_cot_questions`` is the question stream of GraphCoTWorkload: "Which item is linked from
  all of: a; b?" over 2-4 source nodes drawn with a power-law skew; questions recur either at the
  reference generator's measured rate (a stationary stream) or drawn from a fixed pool (as
  generate_workload picks clusters with replacement, workload.cpp:216-225).
* ``scripted_replies`` is the ScriptedProvider trace (scripted.hpp:12-17) of those sessions in the
  Rule agent's formats (rule.cpp:156-236): classify "no" -> per source node "Missing: vertex
  chunks for: <id>" + an action printing NodeInfo(RetrieveNode("<id>")) -> "Finish: <first id>".
"""
from __future__ import annotations

import json
import random

import numpy as np

_ADJ = ("umber", "cobalt", "ivory", "sable", "viridian", "amber", "russet", "pewter", "indigo",
        "maroon", "ochre", "teal", "slate", "coral", "fawn", "lilac")
_NOUN = ("lattice", "widget", "gasket", "spindle", "crucible", "bobbin", "ratchet", "gimbal",
         "flange", "tumbler", "sprocket", "mandrel", "ferrule", "plinth", "luggage", "brazier")
_BRAND = ("acme", "orion", "zephyr", "halcyon", "vertex", "quanta")
_CAT = ("tools", "kitchen", "garden", "office", "sport", "audio")


def _splitmix(seed, k0, count):
    """Outputs k0+1 .. k0+count of the splitmix64 stream seeded with `seed` (vectorised)."""
    with np.errstate(over="ignore"):
        k = np.arange(k0 + 1, k0 + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def node_id(i):
    return "v%07d" % i


def powerlaw_graph_jsonl(n_nodes, edges_per_node, seed, path):
    """Write the synthetic power-law graph as JSONL (graph_store.cpp:38-90 format)."""
    if n_nodes < 2:
        raise ValueError("synthetic graph needs at least 2 nodes")
    is_user = (np.arange(n_nodes) % 10) == 9
    n_items = int((~is_user).sum())
    xs = _splitmix(seed, 0, n_items)
    ex = _splitmix(seed, n_items, n_nodes * edges_per_node)
    u = (ex >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    d = (float(n_nodes) * u * u * u).astype(np.uint64)
    d = np.minimum(d, np.uint64(n_nodes - 1)).astype(np.int64)
    src = np.repeat(np.arange(n_nodes, dtype=np.int64), edges_per_node)
    d = np.where(d == src, (d + 1) % n_nodes, d)
    etype = np.where((ex & np.uint64(3)) == np.uint64(3), "viewed", "linked")
    lines = []
    j = 0
    for i in range(n_nodes):
        nid = node_id(i)
        if is_user[i]:
            lines.append('{"kind":"node","id":"%s","type":"user","attrs":{"name":"user %s"}}\n'
                         % (nid, nid))
        else:
            x = int(xs[j])
            j += 1
            lines.append('{"kind":"node","id":"%s","type":"item","attrs":{"brand":"%s",'
                         '"category":"%s","price":%d,"title":"%s %s %s"}}\n'
                         % (nid, _BRAND[(x >> 32) % 6], _CAT[(x >> 40) % 6], 1 + (x >> 16) % 999,
                            _ADJ[x % 16], _NOUN[(x >> 8) % 16], nid))
    ids = [node_id(i) for i in range(n_nodes)]
    for s, t, et in zip(src.tolist(), d.tolist(), etype.tolist()):
        lines.append('{"kind":"edge","src":"%s","dst":"%s","etype":"%s"}\n' % (ids[s], ids[t], et))
    with open(path, "w", encoding="utf-8") as f:
        f.writelines(lines)
    return path


def graph_cot_questions(n_nodes, n_queries, seed=0, min_hops=2, max_hops=4, skew=2.5,
                        question_pool=0, repeat_frac=0.0, repeat_window=256):
    """[(session id, [source node indices], question text)] of GraphCoTWorkload.

    question_pool > 0: every question is drawn with replacement from that many candidates.
    repeat_frac > 0 (no pool): a stationary stream -- each question repeats one of the previous
    `repeat_window` questions with probability repeat_frac, else it is fresh.  The reference's
    own generator repeats 22% of its questions (generate_workload(7, 1024, 0.5) on synth_graph(7,
    5000): 799 unique of 1024).  Either way the draws are sequential, so the first k questions do
    not depend on n_queries."""
    rnd = random.Random(seed)
    pool = []
    for _ in range(question_pool):
        m = rnd.randint(min_hops, max_hops)
        pool.append([min(n_nodes - 1, int(n_nodes * rnd.random() ** skew)) for _ in range(m)])
    out, hist = [], []
    for q in range(n_queries):
        if pool:
            src = list(pool[rnd.randrange(len(pool))])
        elif repeat_frac > 0 and hist and rnd.random() < repeat_frac:
            recent = hist[-repeat_window:]
            src = list(recent[rnd.randrange(len(recent))])
        else:
            m = rnd.randint(min_hops, max_hops)
            src = [min(n_nodes - 1, int(n_nodes * rnd.random() ** skew)) for _ in range(m)]
        hist.append(src)
        ids = [node_id(v) for v in src]
        out.append((f"q{q:05d}", src, "Which item is linked from all of: " + "; ".join(ids) + "?"))
    return out


def classify_reply():
    return "no\n"


def missing_reply(nid):
    return "Missing: vertex chunks for: " + nid + "\n"


def action_reply(nid):
    return f'```\nprint(NodeInfo(RetrieveNode("{nid}")))\n```\n'


def finish_reply(nid):
    return "Finish: " + nid + "\n"


def scripted_replies(sessions):
    """ScriptedProvider trace lines {session, agent, step, text} for GraphCoTWorkload sessions
    [(sid, sources, question)]."""
    out = []
    for sid, src, _ in sessions:
        ids = [node_id(v) for v in src]
        out.append({"session": sid, "agent": "classification", "step": 0, "text": classify_reply()})
        for r, nid in enumerate(ids):
            out.append({"session": sid, "agent": "reasoning", "step": r, "text": missing_reply(nid)})
            out.append({"session": sid, "agent": "action", "step": r, "text": action_reply(nid)})
        out.append({"session": sid, "agent": "reasoning", "step": len(ids),
                    "text": finish_reply(ids[0])})
    return out


def write_jsonl(rows, path):
    with open(path, "w", encoding="utf-8") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    return path
