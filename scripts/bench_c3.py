"""C3: high-throughput multi-agent Graph-CoT workload (classification / reasoning / action agents),
512 concurrent queries, four-tier priority eviction under a constrained KV pool (BASELINE.json
configs[2]).  Runs the engine (Llama-3-8B shape by default) and replays every prefill and
set_tier, in order, into the reference's own KvCacheState (oracle/_ref): the hit/miss/eviction
counters and the final resident snapshot must be identical (bit-exact cache decisions at scale).

usage: python scripts/bench_c3.py [--lanes 512] [--cap 512] [--rotations 24] [--layers 32]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2511_01633_b200 as glmx  # noqa: E402
from oracle import kv_prefill_inputs  # noqa: E402
from paper_2511_01633_b200 import workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lanes", type=int, default=512)
ap.add_argument("--cap", type=int, default=512)
ap.add_argument("--rotations", type=int, default=24)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--nodes", type=int, default=5000)
ap.add_argument("--policy", type=int, default=glmx.PRIORITY)
ap.add_argument("--sequential", action="store_true", help="no host pipelining")
ap.add_argument("--dump", default=None, help="write the bookkeeping op log (pickle) here")
ap.add_argument("--gemm-tune-tokens", type=int, default=32768,
                help="cuBLAS algorithm table up to this many batch tokens (0 = cublasGemmEx default)")
args = ap.parse_args()

cfg = glmx.ModelConfig(n_layers=args.layers, d_model=4096, n_heads=32, n_kv_heads=8,
                       head_dim=128, d_ff=14336, vocab=128256, seed=0)
g = glmx.PropertyGraph.synth_powerlaw(args.nodes, 8, seed=7, device=0)
ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
model = glmx.Model(cfg, device=0)
if args.gemm_tune_tokens > 0:
    model.tune_gemms(args.gemm_tune_tokens)
kv = glmx.KvCacheState(args.cap, 16, args.policy, device=0, n_layers=cfg.n_layers, n_kv_heads=8,
                       head_dim=128, headroom_pages=args.lanes * 48)
eng = glmx.Engine(model, kv, max_requests=args.lanes, max_batch_tokens=args.lanes * 600,
                  max_decode=8, max_context=8192)
wl = W.GraphCoTWorkload(eng, ret, n_queries=args.lanes * 2, lanes=args.lanes, seed=7,
                        question_pool=args.lanes, node_index=glmx.NodeIndex(g))

# record every bookkeeping op in order: prefills (via prefill_async) and finish() set_tiers
log = []
orig_prefill = wl.prefill_async


def rec_prefill(calls):
    # the reference's run_step order: each call's prefill, then finish()'s set_tier for a Finish
    for c in calls:
        log.append(("p", kv_prefill_inputs(c.segments), c.session.sid))
        if c.is_finish:
            log.append(("t", c.session.sid, 1, 2))
    return orig_prefill(calls)


wl.prefill_async = rec_prefill
eng.set_profiling(1)
t0 = time.perf_counter()
tokens = computed = fwd = 0.0
finished = 0
rots = (wl.rotation() for _ in range(args.rotations)) if args.sequential else wl.rotations(args.rotations)
if args.sequential:
    orig_rot_prefill = wl.prefill

    def rec_prefill_sync(calls, packed=None):
        for c in calls:
            log.append(("p", kv_prefill_inputs(c.segments), c.session.sid))
            if c.is_finish:
                log.append(("t", c.session.sid, 1, 2))
        return orig_rot_prefill(calls, packed)
    wl.prefill = rec_prefill_sync
for r in rots:
    tokens += r.prompt_tokens
    computed += r.computed_tokens
    finished += r.finished
    fwd += eng.last_timings()["forward"]
wall = time.perf_counter() - t0

ref = oracle.RefKv(oracle.ref(), args.cap, 16, args.policy)
for op in log:
    if op[0] == "p":
        (toks, tiers), sess = op[1], op[2]
        st, rep, ev = ref.prefill(toks, tiers, sess)
        assert st == 0, f"reference raised {st} on a prefill the engine accepted"
    else:
        ref.set_tier(op[1], op[2], op[3])
if args.dump:
    import pickle
    pickle.dump({"log": log, "cap": args.cap, "policy": args.policy, "counters": kv.counters(),
                 "resident": kv.resident_snapshot()}, open(args.dump, "wb"))
kc = kv.counters()
ours = [kc["hits"], kc["misses"]] + kc["evictions_by_tier"]
same_counters = list(ref.counters()) == ours
# residents (id, tier, last_used) and every resident's owner session, plus snapshot_json
ours_res = sorted((a, b, lu) for a, b, lu, _ in kv.resident_snapshot())
same_snapshot = (sorted(ref.resident()) == ours_res and ref.snapshot_json() == kv.snapshot()
                 and all(ref.block_session(b) == kv.block_session(b) for b, _, _ in ours_res))
hits, misses = ours[0], ours[1]
print(json.dumps({
    "config": "C3", "lanes": args.lanes, "kv_capacity_blocks": args.cap, "rotations": args.rotations,
    "policy": "priority" if args.policy == glmx.PRIORITY else "plain_lru", "layers": args.layers,
    "prefills": sum(1 for o in log if o[0] == "p"), "finished_queries": finished,
    "prompt_tokens": tokens, "computed_tokens": computed,
    "prefill_tokens_per_s_device": tokens / (fwd * 1e-3), "wall_s": wall,
    "queries_per_s_wall": finished / wall, "block_hit_rate": hits / max(1, hits + misses),
    "counters": {"hits": hits, "misses": misses, "evictions_by_tier": ours[2:]},
    "residents": len(ours_res),
    "bookkeeping_identical_to_reference": same_counters and same_snapshot,
}), flush=True)
assert same_counters and same_snapshot
