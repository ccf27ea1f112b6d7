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
    p.add_argument("--question-pool", type=int, default=0,
                   help="draw every question with replacement from this many candidates; 0 = the "
                        "stationary stream of --repeat-frac")
    p.add_argument("--repeat-frac", type=float, default=0.22,
                   help="share of questions repeating one of the previous 256 (the reference's "
                        "generate_workload(7, 1024, 0.5) repeats 22%%: 799 unique of 1024)")
    p.add_argument("--cache-warm", type=int, default=64,
                   help="untimed rotations before the warm-up steps that bring the prefix cache "
                        "to its steady state (the value then does not drift with --steps)")
    p.add_argument("--routing", default="mod", choices=["mod", "affinity"],
                   help="query -> GPU: i mod N (reference sharding) or prefix affinity "
                        "(fnv1a(question) mod N: repeated questions stay on one GPU)")
    p.add_argument("--no-decode-merge", dest="decode_merge", action="store_false",
                   help="decode every rotation's rows on their own instead of batching two "
                        "rotations' decode rows into one weight stream per step (continuous "
                        "batching, the default: 181.5 vs 170.3 Graph-CoT queries/s on one B200, "
                        "profiles/r2_decode_merge_ab.json)")
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
    p.add_argument("--no-reuse", action="store_true",
                   help="A/B leg: KV reuse off (cache hits recomputed into scratch pages, same "
                        "bookkeeping and prompts); the metric stays prompt tokens/s")
    return p.parse_args()


def workload_shape(args, ws):
    """(queries per rank, question pool, rotations run) -- identical in both arms.  The pool is
    fixed and the question stream is a prefix-stable draw (synth.graph_cot_questions), so the
    rotations that are timed do not depend on --steps."""
    rotations = args.cache_warm + args.warmup + args.steps
    # queries for every rotation the GPU arm runs: + the per-kernel breakdown steps and the
    # Graph-CoT decode phase (the stream is prefix-stable, so this does not change the timed ones)
    n_q = args.lanes * ((rotations + args.steps + getattr(args, "decode_steps", 0)) // 6 + 2)
    return n_q, args.question_pool, rotations


def bench_config(args, ws, pipelined=True, pool_n=None):
    """The `config` object of the JSON line -- the same for `--impl glmx` and `--impl reference`."""
    return {"workload": "C2: Graph-CoT scripted sessions (classify -> reason/act per hop "
                        "-> finish), synthetic 100k-node power-law graph, top-k=16 vertex "
                        "chunks, Llama-3-8B-shaped random-init bf16, paged KV pool",
            "lanes_per_gpu": args.lanes, "nodes": args.nodes, "k": args.k,
            "question_pool": args.question_pool if pool_n is None else pool_n,
            "question_repeat_frac": args.repeat_frac if args.question_pool == 0 else None,
            "cache_warm_rotations": args.cache_warm,
            "kv_capacity_blocks": args.capacity, "block_tokens": 16, "policy": "priority",
            "l2": "inputs > L2 (16 GB weights + KV pool read every step)",
            "parallelism": f"query-sharded x{ws}", "routing": args.routing,
            "host_pipelining": pipelined,
            **({"kv_reuse": False} if getattr(args, "no_reuse", False) else {})}


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) without an external launcher: re-exec under
    torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    NVML (nvidia_ml_py) polled every 10 ms from a thread, each sample time-stamped, so a short
    timed region (~0.7 s at the default --steps) still gets tens of samples and only samples
    taken between mark() and stop() count.  (nvidia-smi -lms piped into Python is block-buffered:
    its lines arrive in bursts, so the round-2 runs saw one sample per region.)  Falls back to
    nvidia-smi when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, device):
        self.device = device
        self.rows = []  # (monotonic time, sm MHz, reasons bitmask)
        self.t0 = self.t1 = None
        self.proc = None
        self.nvml = None
        self.max_mhz = None
        self.halt = threading.Event()

    def mark(self):
        """The timed region starts: only samples from here on count (the sampler is started
        earlier, so its start-up latency does not eat the samples of a short region)."""
        self.t0 = time.monotonic()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # the CUDA device this rank runs on, whatever CUDA_VISIBLE_DEVICES maps it to
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.nvml = (nv, h)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        while not self.halt.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception:
                return
            self.rows.append((time.monotonic(), sm, rs))
            self.halt.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.max_mhz = float(parts[1])
                rs = 0
                for (_, bit), v in zip(self.REASONS, parts[3:]):
                    if v.lower().startswith("active"):
                        rs |= bit
                # nvidia-smi lines arrive buffered: their read time is not their sample time
                self.rows.append((None, float(parts[0]), rs))

    def stop(self):
        self.t1 = time.monotonic()
        if self.nvml is None and self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.halt.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        self.thread.join(timeout=5)
        t0 = self.t0 if self.t0 is not None else -1e30
        rows = [r for r in self.rows if r[0] is None or t0 <= r[0] <= self.t1]
        if not rows:  # a region shorter than the poll interval: the samples around it
            rows = self.rows[-2:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        sm = sorted(r[1] for r in rows)
        reasons = sorted({n for r in rows for n, bit in self.REASONS if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": self.max_mhz,
                "samples": len(rows), "source": "nvml" if self.nvml else "nvidia-smi",
                "reasons": reasons}


def load_traffic():
    """Per-launch DRAM bytes (dram__bytes_read + dram__bytes_write) of each kernel class from the
    committed ncu launch list of the timed C2 step (profiles/r2_c2_traffic.json, made by
    scripts/gpu_step_traffic.sh -> scripts/launch_summary.py --traffic); {} when absent."""
    for name in ("r2_c2_traffic.json", "r1_c2_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)
        except OSError:
            pass
    return {}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------------------
def load_synth():
    """paper_2511_01633_b200/synth.py loaded by path: the reference arm builds the same workload
    without importing the package (no product library is mapped in that process)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "glmx_synth", os.path.join(ROOT, "paper_2511_01633_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def host_cpu():
    """(threads usable, CPU model line) of this host."""
    cores = os.cpu_count() or 1
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return cores, model


class CpuDecoderSlice:
    """The tensor math of the prefill step on the host cores -- which the reference does not have
    (it only costs it, orchestrator.cpp:131-132) -- restated in fp32 numpy: ONE
    Llama-3-8B decoder layer (RMSNorm, QKV, RoPE-free causal GQA attention over each sampled
    call's full context, O, RMSNorm, SwiGLU MLP) timed on a bounded sample of the rotation's
    computed tokens, scaled to all its computed tokens x 32 layers, plus the lm_head rows of the
    rotation's calls (a 1/16 vocabulary slice, x16).  An extrapolation, labelled as such."""

    SAMPLE_TOKENS = 256

    def __init__(self, seed=0):
        import numpy as np

        rng = np.random.default_rng(seed)
        d, self.H, self.Hkv, self.hd, ff = 4096, 32, 8, 128, 14336
        self.d, self.ff = d, ff

        def w(*shape):
            return rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)

        self.w = {"qkv": w((self.H + 2 * self.Hkv) * self.hd, d), "o": w(d, self.H * self.hd),
                  "gu": w(2 * ff, d), "down": w(d, ff), "lm": w(128256 // 16, d)}
        self.np = np

    def _layer(self, n, ctx):
        np, H, Hkv, hd, d = self.np, self.H, self.Hkv, self.hd, self.d
        x = np.ones((n, d), dtype=np.float32)
        h = x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + 1e-5)
        qkv = h @ self.w["qkv"].T
        q = qkv[:, :H * hd].reshape(n, H, hd)
        k = np.concatenate([np.ones((ctx - n, Hkv, hd), np.float32),
                            qkv[:, H * hd:(H + Hkv) * hd].reshape(n, Hkv, hd)])
        v = np.concatenate([np.ones((ctx - n, Hkv, hd), np.float32),
                            qkv[:, (H + Hkv) * hd:].reshape(n, Hkv, hd)])
        mask = np.arange(ctx)[None, :] <= np.arange(ctx - n, ctx)[:, None]
        att = np.empty((n, H, hd), np.float32)
        for hh in range(H):
            s = (q[:, hh] @ k[:, hh // (H // Hkv)].T) * np.float32(hd ** -0.5)
            s = np.where(mask, s, -np.inf)
            p = np.exp(s - s.max(axis=1, keepdims=True))
            att[:, hh] = (p @ v[:, hh // (H // Hkv)]) / p.sum(axis=1, keepdims=True)
        x = x + att.reshape(n, H * hd) @ self.w["o"].T
        h = x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + 1e-5)
        gu = h @ self.w["gu"].T
        g, u = gu[:, :self.ff], gu[:, self.ff:]
        return x + (g / (1 + np.exp(-g)) * u) @ self.w["down"].T

    def rotation_seconds(self, calls):
        """calls [(session, actor, cached, computed)] -> (seconds, description)."""
        np = self.np
        total = sum(c[3] for c in calls)
        sample, got = [], 0
        for c in sorted(calls, key=lambda c: -c[3]):  # the rotation's largest calls first
            if got >= self.SAMPLE_TOKENS or c[3] == 0:
                break
            n = min(c[3], self.SAMPLE_TOKENS - got)
            sample.append((n, c[2] + c[3]))  # the last n tokens of the call, full context
            got += n
        t0 = time.perf_counter()
        for n, ctx in sample:
            self._layer(n, ctx)
        t_layer = time.perf_counter() - t0
        t1 = time.perf_counter()
        np.ones((len(calls), self.d), np.float32) @ self.w["lm"].T
        t_lm = (time.perf_counter() - t1) * 16
        secs = (t_layer / max(1, got)) * total * 32 + t_lm
        return secs, (f"1 layer x {got} sampled tokens {t_layer:.3f}s -> x{total} computed tokens "
                      f"x32 layers, lm_head {len(calls)} rows {t_lm:.3f}s")


def reference_rotations(args, ws, rank, steps, warm):
    """The reference's CPU path over this bench's workload, rotation by rotation: its own
    PropertyGraph::load of the synthetic graph JSONL, Orchestrator + ScriptedProvider (the same
    questions and replies as the GPU arm, rank `rank`'s shard), KvCacheState (capacity, priority)
    and Retriever (node_info k, RetrieveNode over its VectorIndex) -- oracle/_ref, timed exactly
    -- plus the prefill tensor math it lacks (CpuDecoderSlice, extrapolated).  `warm` untimed
    rotations first (cache warm + warm-up, as the GPU arm).  Returns per-step dicts."""
    import oracle

    synth = load_synth()
    tag = f"{os.getpid()}_{args.nodes}_{args.seed}"
    gpath = synth.powerlaw_graph_jsonl(args.nodes, 8, args.seed, f"/tmp/glmx_c2_graph_{tag}.jsonl")
    n_q, pool_n, _ = workload_shape(args, ws)
    sessions = synth.graph_cot_questions(args.nodes, n_q * ws, args.seed, question_pool=pool_n,
                                         repeat_frac=args.repeat_frac)[rank::ws]
    tpath = synth.write_jsonl(synth.scripted_replies(sessions), f"/tmp/glmx_c2_trace_{tag}.jsonl")
    run = oracle.RefScriptedRun(oracle.RefGraph(path=gpath), tpath,
                                [{"id": sid, "text": q} for sid, _, q in sessions], args.lanes,
                                args.capacity, 0, args.k)
    for _ in range(warm):
        run.rotation()
    dec = CpuDecoderSlice(args.seed)
    out = []
    for _ in range(steps):
        t0 = time.perf_counter()
        calls = run.rotation()
        t_book = time.perf_counter() - t0
        t_math, desc = dec.rotation_seconds(calls)
        out.append({"tokens": sum(c[2] + c[3] for c in calls),
                    "computed": sum(c[3] for c in calls), "calls": len(calls),
                    "t_book": t_book, "t_math": t_math, "desc": desc})
    for p in (gpath, tpath):
        try:
            os.remove(p)
        except OSError:
            pass
    return out


def summarize_reference(rows):
    tok = sum(r["tokens"] for r in rows)
    t_book = sum(r["t_book"] for r in rows)
    t_math = sum(r["t_math"] for r in rows)
    value = tok / (t_book + t_math)
    cores, model = host_cpu()
    sample = (f"{len(rows)} rotations ({sum(r['calls'] for r in rows)} calls, {tok} prompt tokens, "
              f"{sum(r['computed'] for r in rows)} computed): reference Orchestrator + "
              f"ScriptedProvider + KvCacheState + Retriever (oracle/_ref) {t_book:.3f}s timed, + "
              f"fp32 numpy prefill math {t_math:.2f}s (per rotation: {rows[-1]['desc']}); "
              f"host: {cores} threads, {model}")
    return value, cores, sample


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path on this bench's workload (rank 0 only)."""
    if rank != 0:
        return
    rows = reference_rotations(args, ws, rank, args.steps, args.cache_warm + args.warmup)
    value, cores, sample = summarize_reference(rows)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "scaling": "weak", "dtype": "f32", "data": "synthetic",
           "config": bench_config(args, ws, not args.no_pipeline),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "cache_hit_token_frac": 1 - sum(r["computed"] for r in rows) / max(1, sum(r["tokens"] for r in rows))}
    print(json.dumps(out))


# ------------------------------------------------------------------------------------------
def standalone_kernels(glmx, g, ret, peaks, tc_peak_burst):
    """K1, K2 and K3 timed alone on synthetic inputs of their large-batch / long-context regimes."""
    import random

    import torch

    import paper_2511_01633_b200.attention as A
    out = {}
    rnd = random.Random(65536)
    nodes = [rnd.randrange(g.node_count()) for _ in range(65536)]
    ret.chunk_build_device(nodes)
    runs = [ret.chunk_build_device(nodes) for _ in range(7)]  # median of 7 builds
    tb, tt, _ = runs[0]
    ms = sorted(r[2] for r in runs)[len(runs) // 2]
    deg = sum(g.total_degree(i) for i in nodes)
    by = 8 * len(nodes) + 8 * deg + 2 * tb + 20 * tt
    out["K1"] = {"workload": "65536 chunks (k=16) of the bench graph, median of 7 builds", "ms": ms,
                 "achieved": by / ms / 1e6, "unit": "GB/s", "frac": by / ms / 1e6 / peaks["hbm_gbs"],
                 "note": "latency/issue-bound byte work (text render + table-driven tokens): ncu in profiles/r2_ncu_k1_v4.txt"}
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
    # K2 in its bandwidth regime with inputs larger than L2 (402 MB per launch)
    from paper_2511_01633_b200.ops import rope_kv_append
    T, L = 16384, 4
    n_pages = T // B + 8
    pool = torch.zeros((n_pages, L, 2, Hkv, B, hd), dtype=torch.bfloat16, device="cuda")
    qkv = torch.randn((T, (H + 2 * Hkv) * hd), device="cuda").to(torch.bfloat16)
    pos = torch.randint(0, 8192, (T,), dtype=torch.int32, device="cuda")
    perm = torch.randperm(n_pages, device="cuda")[: T // B]
    tok = torch.arange(T, device="cuda")
    slot = (perm[tok // B] * B + tok % B).to(torch.int64)
    q_out = torch.empty((T, H, hd), dtype=torch.bfloat16, device="cuda")
    rope_kv_append(qkv, pos, slot, pool, q_out, H, Hkv, layer=1, reps=3)
    ms = rope_kv_append(qkv, pos, slot, pool, q_out, H, Hkv, layer=1, reps=20)
    by = T * ((H + 2 * Hkv) * hd * 2 + H * hd * 2 + 2 * Hkv * hd * 2)
    out["K2"] = {"workload": "16384 tokens (inputs 402 MB > L2), Llama-3-8B heads", "ms": ms,
                 "achieved": by / ms / 1e6, "unit": "GB/s", "frac": by / ms / 1e6 / peaks["hbm_gbs"]}
    del pool, qkv, q_out
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
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
        # the communicator set-up (rings / NVLS over NVSwitch) goes to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
    if args.no_reuse:
        eng.set_reuse(False)
    # enough queries (per rank) that every lane stays busy through the timed rotations
    n_q, pool_n, _ = workload_shape(args, ws)
    nidx = glmx.NodeIndex(g)  # RetrieveNode: device VectorIndex + retrieval LRU (K5)
    wl = GraphCoTWorkload(eng, ret, n_queries=n_q * ws, lanes=args.lanes, seed=args.seed,
                          question_pool=pool_n, node_index=nidx, repeat_frac=args.repeat_frac)
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

    # steady state: the cache-warm rotations, then the warm-up steps (both untimed); the clock
    # sampler starts during the warm-up
    sampler = ClockSampler(local)
    for i, _ in enumerate(rotations(args.cache_warm + args.warmup)):
        if i == args.cache_warm:
            sampler.start()
    if args.warmup <= 0:
        sampler.start()
    # the timed steps carry one CUDA event pair per forward (profiling 1: the forward's device
    # time); the per-kernel-category breakdown is taken over the same number of further steps
    # right after (profiling 2: an event pair around every kernel group), so its event records
    # stay out of the headline
    eng.set_profiling(1)
    peer0 = kv.peer_hits() if px is not None else 0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    prof_range = os.environ.get("GLMX_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    tokens = computed = cached = calls = chunks = finished = 0
    fwd_ms = 0.0
    io0 = eng.io_bytes(), g.io_bytes()
    chunk_ms = 0.0
    k1_bytes = 0
    k5_launches = 0
    k5_ms = 0.0
    k1_rotations = 0
    for r in rotations(args.steps):
        fwd_ms += eng.last_timings()["forward"]
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
    ev1.record()
    torch.cuda.synchronize()
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    wall_ms = ev0.elapsed_time(ev1)
    # host<->device bytes of the timed steps, counted by the engine (packed batch metadata up,
    # greedy ids down) and the graph (RetrieveNode query embeddings + K1 node ids up, winners +
    # chunk bytes / offsets / token ids / spans down)
    io1 = eng.io_bytes(), g.io_bytes()
    h2d = (io1[0][0] - io0[0][0]) + (io1[1][0] - io0[1][0])
    d2h = (io1[0][1] - io0[0][1]) + (io1[1][1] - io0[1][1])


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
    # per-kernel-category breakdown (device time of each kernel group + its algorithmic work),
    # over as many prefill rotations as were timed, after the Graph-CoT phase
    eng.set_profiling(2)
    cat_ms = {"attention": 0.0, "kv_append": 0.0, "gemm": 0.0, "elementwise": 0.0}
    work = {"attn_flops": 0.0, "attn_bytes": 0.0, "append_bytes": 0.0, "linear_flops": 0.0}
    bd_fwd_ms = 0.0
    k2_big_ms = k2_big_bytes = 0.0
    for r in rotations(args.steps):
        tm = eng.last_timings()
        bd_fwd_ms += tm["forward"]
        for k in cat_ms:
            cat_ms[k] += tm[k]
        wk = eng.last_work()
        for k in work:
            work[k] += wk[k]
        if wk["computed_tokens"] >= 2048:  # K2 in its bandwidth regime (large prefill batches)
            k2_big_ms += tm["kv_append"]
            k2_big_bytes += wk["append_bytes"]
    eng.set_profiling(0)
    tm = dict(cat_ms, forward=bd_fwd_ms)
    wk = work
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
        kernels.append({"kernel": "K1 chunk_build (length+scan over the ranked adjacency, render+tokenize)",
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
    # embed + RoPE table, 5 per layer (RMSNorm, K2, K3, RMSNorm, SwiGLU), final norm + split argmax
    launches_per_fwd = 2 + 5 * n_layers + 3
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(args, ws, pipelined, pool_n),
        "gemm_algorithms": {"tuned_up_to_tokens": args.gemm_tune_tokens,
                            "buckets_with_winner": gemm_tuned, "tune_s": round(t_tune, 2)},
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
             "decode": ("continuous batching: two rotations' decode rows per weight stream"
                        if args.decode_merge else "each rotation's rows alone"),
             "n_gpus": ws}
            if dq_ms > 0 else None),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "roofline": roof,
        "kernels": kernels,
        # own kernels in the timed region: the forward's per step (K3's combine pass, launched
        # only for split items, not counted), 3 K1 launches per rotation that built chunks
        # (length+scan, regular chunks, irregular chunks), one K5 scan per rotation that probed
        # the index (cuBLAS GEMMs are library launches, not counted)
        "gpu_launches": int(args.steps * launches_per_fwd + 3 * k1_rotations + k5_launches),
        "clocks": clocks,
    }
    if ws == 1 and not args.no_cpu_baseline:
        # the reference's CPU path on a bounded sample of the same rotations (3 timed rotations
        # after the same warm-up), on this host's cores
        rows = reference_rotations(args, ws, rank, 3, args.cache_warm + args.warmup)
        v, cores, sample = summarize_reference(rows)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                               "sample": sample}
    print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
