"""Timing check of the retrieval / prefill overlap against the reference's pipeline law
(pipeline.hpp:33-38): pipelined_total = P + D1 + max(R, D2), serial_total = P + D1 + R + D2.

In the Graph-CoT rotation (workload.GraphCoTWorkload.rotation) the action's RetrieveNode -> NodeInfo
work (K5 nearest scan + K1 chunk build on the graph's CUDA stream, in a second host thread) does not
depend on the rotation's prefill (replies are scripted), so it runs under that prefill: the work it
hides behind (the law's D2) is the prefill forward, and D1 = 0 (no decode before the call).  Per
rotation the law then predicts
    serial    = H + P + R
    pipelined = H + max(P, R)          (H: the rotation's other host work, identical in both)
The script runs the same C2 rotations twice from the same cache state -- overlap off (retrieval
after the prefill, in advance()) and on -- and compares the measured pipelined wall time with the
law's prediction from the serial run's measured P and R, plus the share of each retrieval interval
that lies inside its rotation's prefill interval.

usage: python scripts/pipeline_law.py [--layers 32] [--rotations 12] [--warm 24] > out.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.workload import GraphCoTWorkload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--lanes", type=int, default=64)
ap.add_argument("--rotations", type=int, default=12)
ap.add_argument("--warm", type=int, default=24)
args = ap.parse_args()

cfg = glmx.ModelConfig(n_layers=args.layers, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                       d_ff=14336, vocab=128256)
g = glmx.PropertyGraph.synth_powerlaw(100_000, 8, seed=0, device=0)
model = glmx.Model(cfg, device=0)
model.tune_gemms(12288)


def run(overlap):
    kv = glmx.KvCacheState(16384, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                           n_kv_heads=8, head_dim=128, headroom_pages=4096)
    eng = glmx.Engine(model, kv, max_requests=args.lanes, max_batch_tokens=args.lanes * 1024,
                      max_decode=8, max_context=8192)
    ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
    n_q = args.lanes * ((args.warm + args.rotations) // 6 + 2)
    wl = GraphCoTWorkload(eng, ret, n_queries=n_q, lanes=args.lanes, seed=0,
                          node_index=glmx.NodeIndex(g), repeat_frac=0.22, overlap_retrieval=overlap)
    spans = {"prefill": [], "retrieve": []}
    pre, rab = wl.prefill, wl._retrieve_and_build

    def timed(tag, fn):
        def w(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                spans[tag].append((t0, time.perf_counter()))
        return w

    wl.prefill = timed("prefill", pre)
    wl._retrieve_and_build = timed("retrieve", rab)
    for _ in range(args.warm):
        wl.rotation()
    eng.set_profiling(1)
    rows = []
    for _ in range(args.rotations):
        for v in spans.values():
            v.clear()
        t0 = time.perf_counter()
        r = wl.rotation()
        wall = (time.perf_counter() - t0) * 1e3
        (p0, p1), = spans["prefill"]
        rs = spans["retrieve"]
        R = sum(b - a for a, b in rs) * 1e3
        inside = sum(max(0.0, min(b, p1) - max(a, p0)) for a, b in rs) * 1e3
        rows.append({"wall_ms": wall, "P_ms": (p1 - p0) * 1e3, "R_ms": R,
                     "R_inside_P_ms": inside, "P_forward_device_ms": eng.last_timings()["forward"],
                     "R_device_ms": r.chunk_ms + r.retrieve_ms, "chunks": r.chunks,
                     "prompt_tokens": r.prompt_tokens})
    eng.close()
    kv.close()
    return rows


def mean(rows, k):
    return sum(r[k] for r in rows) / len(rows)


ser = run(False)
pip = run(True)
P, R = mean(ser, "P_ms"), mean(ser, "R_ms")
H = mean(ser, "wall_ms") - P - R
out = {
    "law": "pipeline.hpp:33-38 pipelined_total = P + D1 + max(R, D2); here D1 = 0, D2 = the "
           "rotation's prefill (P), H = other host work of the rotation",
    "rotations": args.rotations, "lanes": args.lanes, "layers": args.layers,
    "serial": {"wall_ms": mean(ser, "wall_ms"), "P_ms": P, "R_ms": R, "H_ms": H,
               "R_device_ms": mean(ser, "R_device_ms"),
               "law_serial_total_ms": H + P + R},
    "pipelined": {"wall_ms": mean(pip, "wall_ms"), "P_ms": mean(pip, "P_ms"),
                  "R_ms": mean(pip, "R_ms"), "R_device_ms": mean(pip, "R_device_ms"),
                  "R_inside_P_frac": sum(r["R_inside_P_ms"] for r in pip) /
                  max(1e-9, sum(r["R_ms"] for r in pip)),
                  "law_pipelined_total_ms": H + max(P, R)},
    "saving_ms": {"measured": mean(ser, "wall_ms") - mean(pip, "wall_ms"),
                  "law": min(P, R)},
    "per_rotation": {"serial": ser, "pipelined": pip},
}
print(json.dumps(out))
