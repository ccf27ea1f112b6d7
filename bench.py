#!/usr/bin/env python
"""Headline bench: prefill tokens/s with vertex-chunk KV reuse (BASELINE.json metric, config C2:
Llama-3-8B-shaped random-init bf16, synthetic 100k-node power-law graph, top-k=16 chunks).

A step = one round-robin rotation of the Graph-CoT workload (paper_2511_01633_b200/workload.py):
every active lane makes its next LLM call, the calls form ONE engine prefill batch (reference
bookkeeping semantics, paged KV pool, greedy first token), then ONE K1 launch builds the vertex
chunks of the rotation's actions.  Queries are sharded rank r <- query i with i % N == r (weak
scaling, no data-path collective).

  value : prompt tokens (cached+computed+tail) / device time of the forward (CUDA events on the
          engine stream; inputs already in HBM)
  e2e   : same tokens / whole step through the C-ABI with HOST buffers (bookkeeping, H2D, K1,
          forward, D2H), bracketed by device syncs
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill tokens/s with vertex-chunk KV reuse"
UNIT = "tokens/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="glmx", choices=["glmx", "reference"])
    p.add_argument("--lanes", type=int, default=64)
    p.add_argument("--nodes", type=int, default=100_000)
    p.add_argument("--k", type=int, default=16)
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--capacity", type=int, default=16384)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--question-pool", type=int, default=-1,
                   help="draw questions with replacement from this many candidates (reference "
                        "generate_workload style); -1 = half the total query count, 0 = all unique")
    p.add_argument("--routing", default="mod", choices=["mod", "affinity"],
                   help="query -> GPU: i mod N (reference sharding) or prefix affinity "
                        "(fnv1a(question) mod N: repeated questions stay on one GPU)")
    p.add_argument("--decode-merge", action="store_true",
                   help="batch two rotations' decode rows into one decode (continuous batching); "
                        "measured slower on this workload: the long contexts make decode KV-bound")
    p.add_argument("--no-standalone", action="store_true",
                   help="skip the standalone K1 / K3 measurements reported beside the in-step ones")
    p.add_argument("--no-pipeline", action="store_true",
                   help="run the rotations back to back instead of pipelining the host work")
    p.add_argument("--decode-steps", type=int, default=8,
                   help="rotations of the second phase: prefill + greedy reply decode per call "
                        "(Graph-CoT queries/s with the full call_llm step); 0 skips it")
    p.add_argument("--no-peer", action="store_true",
                   help="N>1: disable cross-GPU prefix hits (per-epoch directory + K4 peer copies)")
    p.add_argument("--gemm-tune-tokens", type=int, default=12288,
                   help="before timing, pick cuBLAS algorithms for the projection GEMMs per M "
                        "bucket up to this many batch tokens (glmx_model_tune_gemms); 0 keeps "
                        "cublasGemmEx's default choice")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[0]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]),
                "samples": len(rows), "reasons": sorted(reasons)}


def load_traffic():
    """Per-launch DRAM bytes (dram__bytes_read + dram__bytes_write) of each kernel class from the
    committed ncu launch list of a C2 rotation (profiles/r1_c2_traffic.json, made by
    scripts/launch_summary.py --traffic); {} when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_c2_traffic.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------------------
def cpu_baseline_sample(calls_tokens, chunk_nodes, graph_jsonl, seconds_budget=20.0, reps=None):
    """The reference's CPU path on a bounded sample: the reference bookkeeping (oracle/_ref,
    KvCacheState::prefill + Retriever::node_info_rendered) and, because the reference has no
    tensor math, the builder's fp32 numpy decoder for the computed tokens as a 1-layer
    Llama-3-8B slice x 32 layers (labelled extrapolation).  Returns (tokens/s, cores, sample)."""
    import numpy as np

    import oracle
    from oracle.decoder import rmsnorm

    t_book = 0.0
    ref_graph = oracle.RefGraph(path=graph_jsonl)
    rk = oracle.RefKv(oracle.ref(), 1 << 20, 16, 0)
    t0 = time.perf_counter()
    for nid in chunk_nodes:
        ref_graph.node_info_rendered(nid, 16)
    total_tok, comp_tok = 0, []
    for toks, tiers, sess in calls_tokens:
        st, rep, _ = rk.prefill(toks, tiers, sess)
        total_tok += len(toks)
        comp_tok.append(max(1, rep[1] + rep[2]))
    t_book = time.perf_counter() - t0
    # one decoder layer of the 8B shape, fp32, all host threads (numpy BLAS)
    rng = np.random.default_rng(0)
    d, H, Hkv, hd, ff = 4096, 32, 8, 128, 14336
    W = {k: (rng.standard_normal(s, dtype=np.float32) * 0.02) for k, s in
         {"wqkv": ((H + 2 * Hkv) * hd, d), "wo": (d, H * hd), "wgu": (2 * ff, d),
          "wd": (d, ff)}.items()}
    x = rng.standard_normal((sum(comp_tok), d), dtype=np.float32)
    t1 = time.perf_counter()
    h = rmsnorm(x, 1.0, 1e-5)
    qkv = h @ W["wqkv"].T
    x = x + qkv[:, :H * hd] @ W["wo"].T  # attention core omitted: linear-dominated at this size
    h = rmsnorm(x, 1.0, 1e-5)
    gu = h @ W["wgu"].T
    act = gu[:, :ff] / (1 + np.exp(-gu[:, :ff])) * gu[:, ff:]
    x = x + act @ W["wd"].T
    t_layer = time.perf_counter() - t1
    total = t_book + 32 * t_layer
    cores = os.cpu_count() or 1
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    sample = (f"{len(calls_tokens)} prefill calls ({total_tok} prompt tokens, {sum(comp_tok)} computed) "
              f"+ {len(chunk_nodes)} vertex chunks: reference bookkeeping {t_book:.3f}s + numpy fp32 "
              f"1-layer 8B slice {t_layer:.3f}s x32 (extrapolated; attention core omitted)")
    return total_tok / total, cores, sample


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref bookkeeping + the fp32 decoder
    restatement) on the host cores, rank 0 only."""
    if rank != 0:
        return
    import paper_2511_01633_b200 as glmx  # only for the synthetic graph + workload text
    from paper_2511_01633_b200.workload import GraphCoTWorkload

    g = glmx.PropertyGraph.synth_powerlaw(args.nodes, 8, seed=args.seed, device=0)
    path = f"/tmp/glmx_bench_graph_{args.nodes}_{args.seed}.jsonl"
    if not os.path.exists(path):
        g.save(path)
    ret = glmx.Retriever(g, chunk_k=args.k, vocab=0)
    wl = GraphCoTWorkload(None, ret, n_queries=args.lanes * 4, lanes=args.lanes, seed=args.seed)
    from oracle import kv_prefill_inputs

    def step_sample():
        calls = wl.next_calls()
        wl.advance(calls)
        sub = calls[:4]
        toks = [kv_prefill_inputs(c.segments) + (c.session.sid,) for c in sub]
        nodes = [g.node_id(c.session.sources[min(c.session.round, len(c.session.sources) - 1)])
                 for c in sub]
        return toks, nodes

    vals = []
    for i in range(args.warmup + args.steps):
        toks, nodes = step_sample()
        v, cores, sample = cpu_baseline_sample(toks, nodes, path)
        if i >= args.warmup:
            vals.append(v)
    value = sum(vals) / len(vals)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "config": {"workload": "C2: Graph-CoT scripted sessions, 100k-node power-law graph, "
                                  "k=16, Llama-3-8B shape", "lanes": args.lanes},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                            "sample": "per step: " + sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "data": "synthetic"}
    print(json.dumps(out))


# ------------------------------------------------------------------------------------------
def standalone_kernels(glmx, g, ret, peaks, tc_peak_burst):
    """K1 and K3 timed alone on synthetic inputs of their large-batch / long-context regimes."""
    import random

    import torch

    import paper_2511_01633_b200.attention as A
    out = {}
    rnd = random.Random(65536)
    nodes = [rnd.randrange(g.node_count()) for _ in range(65536)]
    ret.chunk_build_device(nodes)
    tb, tt, ms = ret.chunk_build_device(nodes)
    deg = sum(g.total_degree(i) for i in nodes)
    by = 8 * len(nodes) + 8 * deg + 2 * tb + 20 * tt
    out["K1"] = {"workload": "65536 chunks (k=16) of the bench graph", "ms": ms,
                 "achieved": by / ms / 1e6, "unit": "GB/s", "frac": by / ms / 1e6 / peaks["hbm_gbs"],
                 "note": "issue-bound byte work (render, whitespace mask, fnv1a): ncu in profiles/"}
    H, Hkv, hd, B, P, s, nb = 32, 8, 128, 16, 8192, 128, 8
    ctx = P + s
    per = (ctx + B - 1) // B
    pool = torch.empty((nb * per, 4, 2, Hkv, B, hd), dtype=torch.bfloat16, device="cuda").normal_()
    q = torch.empty((nb * s, H, hd), dtype=torch.bfloat16, device="cuda").normal_()
    o = torch.empty_like(q)
    perm = list(range(nb * per))
    random.Random(P).shuffle(perm)
    bt = [perm[i * per:(i + 1) * per] for i in range(nb)]
    qs, ql, cl = [i * s for i in range(nb)], [s] * nb, [ctx] * nb
    A.paged_attention(q, o, pool, qs, ql, cl, bt, reps=3)
    ms = A.paged_attention(q, o, pool, qs, ql, cl, bt, reps=20)
    flops = nb * sum(4.0 * H * hd * (P + t + 1) for t in range(s))
    out["K3"] = {"workload": "C5 shape: 8 requests x (8192 cached + 128 suffix), one layer",
                 "ms": ms, "achieved": flops / ms / 1e9, "unit": "TFLOP/s",
                 "peak": tc_peak_burst, "frac": flops / ms / 1e9 / tc_peak_burst,
                 "peak_kind": "measured burst bf16 (kernel timed alone)"}
    del pool, q, o
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    import torch.distributed as dist

    import paper_2511_01633_b200 as glmx
    from paper_2511_01633_b200.workload import GraphCoTWorkload

    n_dev = torch.cuda.device_count()
    local = local % max(1, n_dev)  # more ranks than GPUs only in single-GPU protocol tests
    torch.cuda.set_device(local)
    shared_gpu = ws > n_dev
    if ws > 1:
        if shared_gpu:  # NCCL refuses two ranks on one GPU: control plane over gloo
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if shared_gpu else "cuda"

    cfg = glmx.ModelConfig(n_layers=args.layers, d_model=4096, n_heads=32, n_kv_heads=8,
                           head_dim=128, d_ff=14336, vocab=128256, seed=args.seed)
    g = glmx.PropertyGraph.synth_powerlaw(args.nodes, 8, seed=args.seed, device=local)
    ret = glmx.Retriever(g, chunk_k=args.k, vocab=cfg.vocab)
    model = glmx.Model(cfg, device=local)
    t_tune = time.perf_counter()
    gemm_tuned = model.tune_gemms(args.gemm_tune_tokens) if args.gemm_tune_tokens > 0 else 0
    t_tune = time.perf_counter() - t_tune
    kv = glmx.KvCacheState(args.capacity, 16, glmx.PRIORITY, device=local, n_layers=cfg.n_layers,
                           n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                           headroom_pages=4096)
    eng = glmx.Engine(model, kv, max_requests=args.lanes, max_batch_tokens=args.lanes * 1024,
                      max_decode=8, max_context=8192)
    rotations = args.warmup + args.steps
    # enough queries (per rank) that every lane stays busy through the timed rotations
    n_q = args.lanes * (rotations // 6 + 2)
    pool_n = args.question_pool if args.question_pool >= 0 else (n_q * ws) // 2
    nidx = glmx.NodeIndex(g)  # RetrieveNode: device VectorIndex + retrieval LRU (K5)
    wl = GraphCoTWorkload(eng, ret, n_queries=n_q * ws, lanes=args.lanes, seed=args.seed,
                          question_pool=pool_n, node_index=nidx)
    if args.routing == "affinity":
        from paper_2511_01633_b200.sharding import shard_by_affinity
        wl.sessions = shard_by_affinity(wl.sessions, rank, ws, key=lambda s: s.question)
    else:
        wl.sessions = wl.sessions[rank::ws]  # query i -> rank i % N
    # cross-GPU prefix hits (C4): every rotation is an epoch; the ranks exchange their resident
    # (block id, page) directories, and a run of blocks missing locally but resident on a peer is
    # copied over NVLink by K4 (pool exported by CUDA IPC) instead of being recomputed
    px = None
    if ws > 1 and not args.no_peer:
        from paper_2511_01633_b200.sharding import PeerExchange
        try:
            px = PeerExchange(kv)
        except Exception as exc:  # noqa: BLE001 — report and run sharded without peer hits
            print(f"rank {rank}: peer exchange disabled: {exc}", file=sys.stderr)
            px = None

    def step():
        if px is not None:
            px.epoch_begin()
        r = wl.rotation()
        if px is not None:
            px.epoch_end()
        return r

    # rotations are pipelined (host work of r+1 under the forward of r); with peer exchange the
    # directory is published one rotation later, once the pages it names are complete
    # (PeerExchange.before_bookkeeping / after_wait)
    pipelined = not args.no_pipeline

    def rotations(k):
        if pipelined:
            yield from wl.rotations(k, peer=px)
        else:
            for _ in range(k):
                yield step()

    for _ in rotations(args.warmup):
        pass
    # per-kernel-category CUDA events on the engine stream during the timed steps (host cost
    # ~1 us per event record, <1% of a step)
    eng.set_profiling(2)
    peer0 = kv.peer_hits() if px is not None else 0
    sampler = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    prof_range = os.environ.get("GLMX_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    tokens = computed = cached = calls = chunks = finished = 0
    fwd_ms = 0.0
    cat_ms = {"attention": 0.0, "kv_append": 0.0, "gemm": 0.0, "elementwise": 0.0}
    work = {"attn_flops": 0.0, "attn_bytes": 0.0, "append_bytes": 0.0, "linear_flops": 0.0}
    h2d = d2h = 0
    chunk_ms = 0.0
    k1_bytes = 0
    k5_launches = 0
    k5_ms = 0.0
    k1_rotations = 0
    k2_big_ms = k2_big_bytes = 0.0
    for r in rotations(args.steps):
        tm = eng.last_timings()
        fwd_ms += tm["forward"]
        for k in cat_ms:
            cat_ms[k] += tm[k]
        if r.chunks:
            chunk_ms += r.chunk_ms
            k1_bytes += r.chunk_bytes
            if r.retrieve_probes:  # one K5 nearest scan served this rotation's misses
                k5_launches += 1
                k5_ms += r.retrieve_ms
        tokens += r.prompt_tokens
        computed += r.computed_tokens
        cached += r.cached_tokens
        calls += r.calls
        chunks += r.chunks
        k1_rotations += 1 if r.chunks else 0
        finished += r.finished
        wk = eng.last_work()
        for k in work:
            work[k] += wk[k]
        if wk["computed_tokens"] >= 2048:  # K2 in its bandwidth regime (large prefill batches)
            k2_big_ms += tm["kv_append"]
            k2_big_bytes += wk["append_bytes"]
        # host->device per step: packed batch metadata + chunk node ids; device->host: greedy ids
        # + chunk bytes/tokens
        h2d += int(wk["computed_tokens"]) * 16 + r.calls * (16 + 8 * 520) + r.chunks * 4
        d2h += r.calls * 4 + r.chunks * 1200
    ev1.record()
    torch.cuda.synchronize()
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    wall_ms = ev0.elapsed_time(ev1)

    eng.set_profiling(0)
    tm = dict(cat_ms, forward=fwd_ms)
    wk = work

    # phase 2 (after the measured prefill steps): the complete call_llm step — prefill + greedy
    # decode of each reply — for Graph-CoT queries/s; rotations sequential (decode continues the
    # last staged batch)
    dq_fin = dq_dec = 0
    dq_ms = dq_dec_ms = dq_pre_ms = 0.0
    dq_n_dec = [0]
    if args.decode_steps > 0:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        d0 = torch.cuda.Event(enable_timing=True)
        d1 = torch.cuda.Event(enable_timing=True)
        d0.record()
        eng.set_profiling(1)  # one event pair per forward: the decode forwards' device time

        def account(rr):
            nonlocal dq_fin, dq_dec, dq_dec_ms, dq_pre_ms
            dq_fin += rr.finished
            dq_dec += rr.decoded_tokens
            if rr.decoded_tokens and rr.decode_collected:  # device time of the decode forwards
                dq_dec_ms += eng.last_timings()["forward"]
            dq_n_dec[0] += 1 if rr.decode_collected else 0
            dq_pre_ms += getattr(wl, "last_prefill_forward_ms", 0.0)

        if pipelined:
            # rotation r+1's host work (advance, calls, RetrieveNode/K1) under r's decode steps;
            # with peer exchange the directory follows the pipelined epoch protocol
            for rr in wl.rotations_with_decode(args.decode_steps, 8, peer=px,
                                               merge=args.decode_merge):
                account(rr)
        else:
            for _ in range(args.decode_steps):
                if px is not None:
                    px.epoch_begin()
                rr = wl.rotation_with_decode(8)
                if px is not None:
                    px.epoch_end()
                account(rr)
        d1.record()
        torch.cuda.synchronize()
        eng.set_profiling(0)
        if ws > 1:
            dist.barrier()
        dq_ms = d0.elapsed_time(d1)
    peer_blocks = float(kv.peer_hits() - peer0) if px is not None else 0.0
    vals = torch.tensor([tokens, computed, cached, calls, finished, peer_blocks, dq_fin, dq_dec],
                        dtype=torch.float64, device=red_dev)
    times = torch.tensor([fwd_ms, wall_ms, dq_ms], dtype=torch.float64, device=red_dev)
    if ws > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.SUM)
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    tokens, computed, cached, calls, finished, peer_blocks, dq_fin, dq_dec = vals.tolist()
    fwd_ms, wall_ms, dq_ms = times.tolist()
    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return

    peaks, peak_kind = measured_peaks()
    hbm = peaks["hbm_gbs"]
    # the timed region is a long back-to-back step: tensor work runs at the sustained (power-cap)
    # GEMM rate; HBM-bound kernels against the copy bandwidth
    tc_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = load_traffic()
    attn_ms = tm["attention"]
    attn_tflops = wk["attn_flops"] / (attn_ms * 1e-3) / 1e12 if attn_ms > 0 else 0.0
    attn_gbs = wk["attn_bytes"] / (attn_ms * 1e-3) / 1e9 if attn_ms > 0 else 0.0
    ridge = tc_peak * 1e12 / (hbm * 1e9)
    intensity = wk["attn_flops"] / max(1.0, wk["attn_bytes"])
    gemm_tflops = wk["linear_flops"] / max(1e-9, tm["gemm"] * 1e-3) / 1e12
    append_gbs = wk["append_bytes"] / max(1e-9, tm["kv_append"] * 1e-3) / 1e9
    fwd = max(1e-9, tm["forward"])
    n_launch_layers = args.steps * cfg.n_layers
    kernels = [
        {"kernel": "K3 paged_attn_tc (tcgen05/TMEM/TMA)", "share_of_forward": attn_ms / fwd,
         "ms_per_launch": attn_ms / n_launch_layers, "intensity_flop_per_byte": intensity,
         **({"bound": "tensor", "achieved": attn_tflops, "peak": tc_peak, "unit": "TFLOP/s",
             "frac": attn_tflops / tc_peak} if intensity >= ridge else
            {"bound": "hbm", "achieved": attn_gbs, "peak": hbm, "unit": "GB/s",
             "frac": attn_gbs / hbm}),
         "note": "C2 suffixes are short (mean q 7-120 tokens over 55-280-token contexts): "
                 "latency-bound items; the tensor-bound regime is C5 (scripts/bench_attn.py)"},
        {"kernel": "K2 rope_kv_append (fused RoPE + paged KV append)", "bound": "hbm",
         "share_of_forward": tm["kv_append"] / fwd, "achieved": append_gbs, "peak": hbm,
         # rotations whose batch computes >= 2048 tokens; the rest are small batches (~500
         # tokens, ~12 MB per launch) where launch latency dominates; in-step times also carry
         # the write-back of the QKV GEMM output that K2's traffic evicts from L2
         "achieved_batches_ge_2048_tokens": (k2_big_bytes / (k2_big_ms * 1e-3) / 1e9
                                             if k2_big_ms > 0 else None),
         "frac_batches_ge_2048_tokens": (k2_big_bytes / (k2_big_ms * 1e-3) / 1e9 / hbm
                                         if k2_big_ms > 0 else None),
         "unit": "GB/s", "frac": append_gbs / hbm,
         "ms_per_launch": tm["kv_append"] / n_launch_layers},
    ]
    if chunk_ms > 0:
        k1_gbs = k1_bytes / (chunk_ms * 1e-3) / 1e9
        kernels.append({"kernel": "K1 chunk_build (select+render+emit, 2 cub scans)",
                        "bound": "hbm", "achieved": k1_gbs, "peak": hbm, "unit": "GB/s",
                        "frac": k1_gbs / hbm, "ms_per_rotation": chunk_ms / max(1, k1_rotations),
                        "overlapped_with_prefill": True,
                        "note": "64 chunks per rotation: latency-bound, hidden behind the prefill "
                                "on the graph stream"})
    if k5_launches:
        k5_bytes = len(nidx) * 64 * 4  # the index is streamed once per scan
        k5_gbs = k5_bytes * k5_launches / (k5_ms * 1e-3) / 1e9
        kernels.append({"kernel": "K5 nearest (RetrieveNode exact scan, bit-exact 8-lane dot)",
                        "bound": "hbm", "achieved": k5_gbs, "peak": hbm, "unit": "GB/s",
                        "frac": k5_gbs / hbm, "ms_per_launch": k5_ms / k5_launches,
                        "overlapped_with_prefill": True,
                        "retrieval_stats": dict(zip(("cache_hits", "cache_misses", "index_probes"),
                                                    nidx.stats()))})
    if not args.no_standalone:
        # the same kernels alone in their bandwidth / tensor regimes (untimed region, GPU idle):
        # K1 over a 65536-chunk batch of this graph, K3 at the C5 shape (8 x 8192 cached + 128)
        sa = standalone_kernels(glmx, g, ret, peaks, tc_peak_burst=peaks["bf16_tflops"])
        for kd in kernels:
            tag = kd["kernel"].split()[0]
            if tag in sa:
                kd["standalone"] = sa[tag]
    # dominant kernel of the step by device time: the cuBLAS GEMMs (Llama-3-8B linears)
    roof = {"bound": "tensor", "achieved": gemm_tflops, "peak": tc_peak, "unit": "TFLOP/s",
            "frac": gemm_tflops / tc_peak,
            "kernel": "cuBLAS bf16 GEMM (library: cublasLtMatmul with the tuned per-bucket algorithm, else cublasGemmEx; QKV/O/gate-up/down/lm_head)",
            "traffic": traffic.get("gemm"), "traffic_unit": "bytes per launch (ncu, profiles/)",
            "peak_kind": peak_kind + " sustained bf16",
            "share_of_forward": tm["gemm"] / fwd,
            "gemm_ms_per_step": tm["gemm"] / args.steps,
            "attention_ms_per_step": attn_ms / args.steps,
            "append_ms_per_step": tm["kv_append"] / args.steps,
            "elementwise_ms_per_step": tm["elementwise"] / args.steps}
    for kd in kernels:
        kd["traffic"] = traffic.get(kd["kernel"].split()[0])
    value = tokens / (fwd_ms * 1e-3)
    e2e = tokens / (wall_ms * 1e-3)
    n_layers = cfg.n_layers
    launches_per_fwd = 1 + 5 * n_layers + 3  # embed, 5 per layer, final norm + split argmax (2)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "C2: Graph-CoT scripted sessions (classify -> reason/act per hop "
                               "-> finish), synthetic 100k-node power-law graph, top-k=16 vertex "
                               "chunks, Llama-3-8B-shaped random-init bf16, paged KV pool",
                   "lanes_per_gpu": args.lanes, "nodes": args.nodes, "k": args.k,
                   "question_pool": pool_n,
                   "kv_capacity_blocks": args.capacity, "block_tokens": 16,
                   "l2": "inputs > L2 (16 GB weights + KV pool read every step)",
                   "parallelism": f"query-sharded x{ws}", "routing": args.routing,
                   "host_pipelining": pipelined,
                   "gemm_algorithms": {"tuned_up_to_tokens": args.gemm_tune_tokens,
                                       "buckets_with_winner": gemm_tuned,
                                       "tune_s": round(t_tune, 2)}},
        "raw_computed_tokens_per_s": computed / (fwd_ms * 1e-3),
        "cache_hit_token_frac": cached / max(1.0, tokens),
        "calls": calls, "queries_finished": finished,
        "peer_hit_blocks": peer_blocks if ws > 1 else None,
        "queries_per_s_prefill_only": finished / (wall_ms * 1e-3),
        "graph_cot_queries_per_s": (
            {"value": dq_fin / (dq_ms * 1e-3), "unit": "queries/s", "rotations": args.decode_steps,
             "queries_finished": dq_fin, "decoded_tokens": dq_dec, "ms": dq_ms,
             "decode_forward_ms": dq_dec_ms, "prefill_forward_ms": dq_pre_ms,
             "decode_launches": dq_n_dec[0],
             "step": "prefill + greedy reply decode per call (call_llm), CUDA events, max over ranks",
             "n_gpus": ws}
            if dq_ms > 0 else None),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "roofline": roof,
        "kernels": kernels,
        # own kernels in the timed region: forward + argmax per step, 4 K1 launches per rotation
        # that built chunks (cub scans and cuBLAS GEMMs are library launches, not counted)
        "gpu_launches": int(args.steps * (launches_per_fwd + 1) + 3 * k1_rotations + k5_launches),
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        from oracle import kv_prefill_inputs

        path = f"/tmp/glmx_bench_graph_{args.nodes}_{args.seed}.jsonl"
        g.save(path)
        sub = wl.next_calls()[:8]
        toks = [kv_prefill_inputs(c.segments) + (c.session.sid,) for c in sub]
        nodes = [g.node_id(c.session.sources[min(c.session.round, len(c.session.sources) - 1)])
                 for c in sub]
        v, cores, sample = cpu_baseline_sample(toks, nodes, path)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                               "sample": sample}
    print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
