"""Regenerates tests/golden/golden.json from the reference itself (oracle/_ref, compiled from
/root/reference/proj).  Run in the build container:  python tests/golden/make_golden.py

Contents (each a known answer the reference produced):
  chain_ids      KvCacheState::chain_ids of ["t0".."t63"], B=16 (cache.cpp:31-40)
  node_info      Retriever::node_info_rendered for every fixture node x k x weight mode x dir
  prefill_kats   SPEC.md:505-516 style cases (cold/warm/shared prefix/self-evict/exhausted)
  fig6           ScriptedProvider run of the Fig. 6 trace (C1): per-session records, final
                 snapshot, and the exact prefill / set_tier call sequence the orchestrator made
  bench_traces   run_bench (RuleProvider, round-robin) call sequences, incl. eviction pressure
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def main():
    L = oracle.ref()
    out = {}
    out["chain_ids"] = [str(x) for x in oracle.ref_chain_ids([f"t{i}" for i in range(64)], 16)]
    g = oracle.RefGraph(path=os.path.join(HERE, "tiny.jsonl"))
    ni = []
    for nid in g.node_ids():
        for k in (0, 1, 2, 8):
            for wm in (0, 1):
                for d in (False, True):
                    ni.append([nid, k, wm, d, g.node_info_rendered(nid, k, wm, d)])
    out["node_info"] = ni
    kats = []

    def run(cap, B, policy, ops):
        kv = oracle.RefKv(L, cap, B, policy)
        res = []
        for toks, tiers, sess in ops:
            st, rep, ev = kv.prefill(toks, tiers, sess)
            res.append([st, list(rep), [str(e) for e in ev]])
        return {"cap": cap, "B": B, "policy": policy,
                "ops": [[t, [list(x) for x in tr], s] for t, tr, s in ops], "results": res,
                "counters": kv.counters(), "resident": [[str(a), b, c] for a, b, c in kv.resident()]}

    t64 = [f"t{i}" for i in range(64)]
    kats.append(run(100, 16, 0, [(t64, [(0, 64, 3)], "s"), (t64, [(0, 64, 3)], "s"),
                                 (t64[:32] + [f"x{i}" for i in range(32)], [(0, 64, 3)], "s")]))
    w24 = [f"w{i}" for i in range(24)]
    kats.append(run(4, 4, 0, [(w24, [(0, 24, 3)], "s"), (w24, [(0, 24, 3)], "s")]))
    kats.append(run(2, 16, 0, [(t64, [(0, 64, 0)], "s")]))
    kats.append(run(8, 4, 0, [(t64[:16], [(0, 6, 0), (6, 16, 3)], "s")]))
    kats.append(run(3, 4, 1, [(w24, [(0, 8, 0), (8, 24, 3)], "s"), (w24[:12], [(0, 12, 1)], "t")]))
    out["prefill_kats"] = kats

    qs = [json.loads(x) for x in open(os.path.join(HERE, "fig6_questions.jsonl"))]
    res, trace = g.run_scripted(os.path.join(HERE, "fig6_trace.jsonl"), qs, 8, 4096, 0, 8, True)
    out["fig6"] = {"sessions": res["sessions"], "kv": res["kv"], "trace": trace}

    bt = []
    for nodes, n, lanes, cap, policy in ((500, 40, 8, 4096, 0), (500, 60, 16, 48, 1),
                                         (500, 60, 16, 96, 0)):
        sg = oracle.RefGraph(synth=(7, nodes))
        try:
            rep, trace = sg.run_bench(seed=7, n=n, ratio=0.5, concurrency=lanes, cap=cap,
                                      policy=policy, glm=True, record=True)
            err = None
        except RuntimeError as e:
            rep, err = None, str(e)
            trace = oracle.trace_lines()
        for t in trace:
            if "evicted" in t:
                t["evicted"] = [str(x) for x in t["evicted"]]
        bt.append({"nodes": nodes, "n": n, "lanes": lanes, "cap": cap, "policy": policy,
                   "report": rep, "error": err, "trace": trace})
    out["bench_traces"] = bt
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote golden.json", os.path.getsize(os.path.join(HERE, "golden.json")), "bytes")


if __name__ == "__main__":
    main()
