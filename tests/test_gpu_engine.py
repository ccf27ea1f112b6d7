"""Prefill/decode engine on the GPU vs the CPU fp32 decoder oracle (oracle/decoder.py) and the
reference bookkeeping.  Tolerances (north star): logits max-abs 2e-2 + rel 1e-2 (bf16 vs fp32);
greedy ids bit-exact (asserted where the oracle's top-1/top-2 margin exceeds the tolerance)."""
import os
import numpy as np
import pytest

import oracle
import paper_2511_01633_b200 as glmx
from oracle.decoder import Decoder, token_ids

pytestmark = pytest.mark.gpu
ATOL, RTOL = 2e-2, 1e-2


def make(cfg, cap=256, headroom=256, max_req=16, max_tok=4096, max_decode=8, max_ctx=4096):
    model = glmx.Model(cfg, device=0)
    kv = glmx.KvCacheState(cap, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                           n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                           headroom_pages=headroom)
    eng = glmx.Engine(model, kv, max_requests=max_req, max_batch_tokens=max_tok,
                      max_decode=max_decode, max_context=max_ctx)
    return model, kv, eng


def check_logits(got, want):
    err = np.abs(got - want)
    tol = ATOL + RTOL * np.abs(want)
    assert np.all(err <= tol), f"max err {err.max():.4g} (max |ref| {np.abs(want).max():.3g})"


def check_greedy(got_ids, logits_ref_rows, want_ids):
    for g, w, lr in zip(got_ids, want_ids, logits_ref_rows):
        if g == w:
            continue
        top = np.sort(lr)[-2:]
        assert top[1] - top[0] <= 2 * (ATOL + RTOL * abs(top[1])), (g, w, top)


@pytest.fixture(scope="module")
def tiny():
    model, kv, eng = make(glmx.TINY)
    return model, kv, eng, Decoder(glmx.TINY, model.export_all())


def words(n, tag="w"):
    return [f"{tag}{i}" for i in range(n)]


def test_prefill_batch_with_shared_prefix(tiny):
    model, kv, eng, dec = tiny
    p = words(70)
    reqs = [glmx.Request(p, [(0, 20, 0), (20, 70, 3)], "a"),
            glmx.Request(p[:48] + words(9, "x"), [(0, 57, 1)], "b"),   # hits a's blocks in-batch
            glmx.Request(words(5, "z"), [(0, 5, 3)], "c"),             # tail only
            glmx.Request(p[:64], [(0, 64, 2)], "d")]                   # fully cached -> recompute last
    reps, first, logits = eng.prefill(reqs, want_logits=True)
    assert [(r.cached_tokens, r.computed_tokens, r.tail_tokens) for r in reps] == [
        (0, 64, 6), (48, 0, 9), (0, 0, 5), (64, 0, 0)]
    refs = [dec.forward(token_ids(r.tokens, model.cfg.vocab))[0] for r in reqs]
    for i in range(len(reqs)):
        check_logits(logits[i], refs[i])
    check_greedy(first, refs, [int(np.argmax(x)) for x in refs])


def test_decode_matches_greedy_oracle(tiny):
    model, kv, eng, dec = tiny
    reqs = [glmx.Request(words(40, "q"), [(0, 40, 3)], "s"),
            glmx.Request(words(17, "r"), [(0, 17, 3)], "t")]
    _, first = eng.prefill(reqs)
    out, last = eng.decode([6, 3], want_logits=True)
    assert [len(o) for o in out] == [6, 3]
    for i, r in enumerate(reqs):
        ids = token_ids(r.tokens, model.cfg.vocab)
        dec.check_greedy(ids, [first[i]] + out[i])


G4 = glmx.ModelConfig(n_layers=2, d_model=512, n_heads=8, n_kv_heads=2, head_dim=128, d_ff=1024,
                      vocab=32000)


def test_decode_gqa4_matches_greedy_oracle():
    """GQA 4:1 (the Llama-3 ratio): decode steps run the CUDA-core decode kernel (K3d) with RoPE +
    K/V append fused in; greedy tokens follow the fp32 oracle, last-step logits within tolerance.
    (K3d against the tcgen05 kernel on the same rows: test_gpu_attention.py.)"""
    model, kv, eng = make(G4)
    dec = Decoder(G4, model.export_all())
    reqs = [glmx.Request(words(40, "q"), [(0, 40, 3)], "s"),
            glmx.Request(words(17, "r"), [(0, 17, 3)], "t"),
            glmx.Request(words(300, "p"), [(0, 300, 3)], "u")]
    _, first = eng.prefill(reqs)
    out, last = eng.decode([6, 3, 5], want_logits=True)
    assert [len(o) for o in out] == [6, 3, 5]
    for i, r in enumerate(reqs):
        dec.check_greedy(token_ids(r.tokens, G4.vocab), [first[i]] + out[i])
    ref_last = dec.forward(token_ids(reqs[0].tokens, G4.vocab) + [first[0]] + out[0][:-1])[0]
    check_logits(last[0], ref_last)


def test_decode_twice_on_one_batch_is_rejected(tiny):
    model, kv, eng, dec = tiny
    eng.prefill([glmx.Request(words(20, "dd"), [(0, 20, 3)], "s")])
    eng.decode([2])
    with pytest.raises(glmx.GlmxError):
        eng.decode([2])


def test_failed_batch_leaves_no_garbage_kv():
    """A batch that fails an engine limit (max_batch_tokens) after its bookkeeping committed:
    the cache keeps the reference's decisions (its blocks stay resident and later count as
    cached), but their pages never got KV -- they are stale and recomputed on next use, so the
    retried requests' logits still match the oracle."""
    model, kv, eng = make(glmx.TINY, max_tok=256)
    dec = Decoder(glmx.TINY, model.export_all())
    a, b = words(200, "fa"), words(96, "fa") + words(104, "fb")
    with pytest.raises(glmx.GlmxError):  # 200 + 104 rows > 256 after both were booked
        eng.prefill([glmx.Request(a, [(0, 200, 3)], "s"), glmx.Request(b, [(0, 200, 3)], "t")])
    assert kv.counters()["misses"] > 0
    for toks in (b, a):
        reps, first, logits = eng.prefill([glmx.Request(toks, [(0, 200, 3)], "u")], want_logits=True)
        assert reps[0].cached_tokens == 192  # bookkeeping: the failed batch's blocks are resident
        check_logits(logits[0], dec.forward(token_ids(toks, glmx.TINY.vocab))[0])
    model.close()


def test_bookkeeping_only_prefill_then_engine_recomputes():
    """glmx_kv_prefill on the device pool (bookkeeping only, no forward) inserts blocks whose pages
    hold no KV; the engine's next prefill over them reports them cached (reference semantics) and
    recomputes their KV instead of attending over the empty pages."""
    model, kv, eng = make(glmx.TINY)
    dec = Decoder(glmx.TINY, model.export_all())
    toks = words(100, "bo")
    kv.prefill(toks, [(0, 100, 3)], "s")
    assert all(p == -1 for _, _, _, p in kv.resident_snapshot())  # stale: no KV yet
    reps, first, logits = eng.prefill([glmx.Request(toks + ["x"], [(0, 101, 3)], "s")],
                                      want_logits=True)
    assert reps[0].cached_tokens == 96
    check_logits(logits[0], dec.forward(token_ids(toks + ["x"], glmx.TINY.vocab))[0])
    assert all(p >= 0 for _, _, _, p in kv.resident_snapshot())
    model.close()


def test_tuned_gemm_algorithms_match_oracle():
    """glmx_model_tune_gemms: after the per-(projection, M bucket) cuBLAS algorithm table is
    filled, prefill batches landing in several buckets (and beyond the tuned range) still match
    the fp32 oracle, and the logits agree with the untuned cublasGemmEx forward."""
    cfg = glmx.ModelConfig(n_layers=2, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128,
                           d_ff=8192, vocab=4096)
    model = glmx.Model(cfg, device=0)
    dec = Decoder(cfg, model.export_all())
    batches = [[glmx.Request(words(n, f"b{n}x{j}"), [(0, n, 3)], f"s{n}{j}") for j in range(k)]
               for n, k in ((150, 1), (300, 2), (520, 3), (700, 4))]

    def run():
        kv = glmx.KvCacheState(512, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                               n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                               headroom_pages=512)
        eng = glmx.Engine(model, kv, max_requests=8, max_batch_tokens=4096, max_decode=2,
                          max_context=1024)
        out = [eng.prefill(b, want_logits=True) for b in batches]
        del eng
        kv.close()
        return out

    base = run()
    n = model.tune_gemms(1600)  # the 2800-token batch stays on cublasGemmEx
    assert 0 <= n <= 4 * 15
    tuned = run()
    # d_model 2048 / d_ff 8192 in bf16 sits above the 2e-2 floor of the small configs: the bar is
    # the untuned forward's own error against the oracle (as in the Llama-shaped slice below)
    for b, (_, f0, l0), (_, f1, l1) in zip(batches, base, tuned):
        for i, r in enumerate(b):
            ids = token_ids(r.tokens, cfg.vocab)
            ref = dec.forward(ids)[0]
            e0, e1 = np.abs(l0[i] - ref), np.abs(l1[i] - ref)
            assert e1.max() <= 1.5 * e0.max() + 1e-2 and e1.mean() <= 1.5 * e0.mean() + 1e-3, (
                e0.max(), e1.max(), e0.mean(), e1.mean())
            assert np.abs(l1[i] - l0[i]).max() <= 2 * e0.max() + 1e-2
            dec.check_greedy(ids, [f1[i]], atol=max(2e-2, float(e0.max())), rtol=0.0)
    model.close()


def test_bookkeeping_matches_reference_under_pressure(ref):
    """Same request stream through the engine (device pool) and the reference KvCacheState:
    identical reports, eviction order and residents, including self-eviction + orphans."""
    model, kv, eng = make(glmx.TINY, cap=6, headroom=64)
    rk = oracle.RefKv(ref, 6, 16, 0)
    rnd = np.random.default_rng(1)
    base = words(64)
    for step in range(12):
        reqs = []
        for j in range(3):
            n = int(rnd.integers(1, 120))
            toks = (base[: int(rnd.integers(0, 64))] + words(n, f"s{step}_{j}_"))[:n]
            cut = int(rnd.integers(0, len(toks) + 1))
            tiers = [t for t in [(0, cut, 0), (cut, len(toks), 3)] if t[0] < t[1]]
            reqs.append(glmx.Request(toks, tiers, f"sess{j}"))
        try:
            reps, _ = eng.prefill(reqs)
        except glmx.CacheExhausted:
            reps = None
        for i, r in enumerate(reqs):
            st, rep, ev = rk.prefill(r.tokens, r.tiers, r.session)
            if reps is None:
                break
            assert st == 0
            assert (reps[i].cached_tokens, reps[i].computed_tokens, reps[i].tail_tokens) == rep
        if reps is None:
            break
        assert [(a, b, c) for a, b, c, _ in kv.resident_snapshot()] == rk.resident()


# The Llama-3-8B shape in bf16 storage is numerically chaotic at the logit level: rounding the
# activations to bf16 at the engine's storage points (Decoder(emulate_bf16=True): h1, qkv, q, k,
# v, P with K3's lazy-max tiles, attn, h2, gu, act, hf) and then perturbing the weights by 1e-7 to
# 1e-6 relative -- the size of fp32 accumulation-order differences over K >= 4096 -- moves the
# logits by max ~0.03-0.047 / mean ~0.005-0.008 and leaves up to ~1% of the 128256 logits outside
# 2e-2 + 1e-2|x|, while the same perturbation moves the plain fp32 forward by ~1e-5
# (scripts/cpu_bf16_sensitivity.py).  No implementation with bf16 storage can meet 2e-2 on every
# logit against an oracle that does not replicate its accumulation order bit for bit.  The test
# therefore measures that chaos floor on the oracle itself, for these very inputs (two 2^-20
# relative weight perturbations, the worse one), and requires the engine to sit inside it: max /
# mean error vs the bf16-emulating oracle within 1.5x the floor, the share of logits within
# 2e-2 / 1e-2 at most 1% below the floor's; plus the fp32 bound (1.5x the fp32-vs-bf16 floor,
# max 0.074 / mean 0.0126).
FLOOR_MAX, FLOOR_MEAN = 0.074, 0.0126


def chaos_floor(cfg, w, ids, ref_bf, seeds=(1, 2), eps=2.0 ** -20):
    worst = (0.0, 0.0, 1.0)
    for seed in seeds:
        rng = np.random.default_rng(seed)

        def pert(m):
            return (m * (1 + eps * rng.standard_normal(m.shape, dtype=np.float32))).astype(np.float32)

        wp = dict(w, layers=[{k: (pert(v) if v.ndim == 2 else v) for k, v in lw.items()}
                             for lw in w["layers"]])
        d = Decoder(cfg, wp, emulate_bf16=True).forward(ids)[0]
        e = np.abs(d - ref_bf)
        worst = (max(worst[0], float(e.max())), max(worst[1], float(e.mean())),
                 min(worst[2], float(np.mean(e <= ATOL + RTOL * np.abs(ref_bf)))))
    return worst


@pytest.mark.slow
def test_llama8b_shape_two_layer_slice():
    cfg = glmx.ModelConfig(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128,
                           d_ff=14336, vocab=128256)
    model, kv, eng = make(cfg, cap=64, headroom=64, max_req=4, max_tok=1024, max_decode=2,
                          max_ctx=1024)
    w = model.export_all()
    dec = Decoder(cfg, w)
    dec_bf = Decoder(cfg, w, emulate_bf16=True)
    p = words(150)
    reqs = [glmx.Request(p, [(0, 40, 0), (40, 150, 3)], "a"),
            glmx.Request(p[:130] + words(30, "y"), [(0, 160, 1)], "b")]
    reps, first, logits = eng.prefill(reqs, want_logits=True)
    assert reps[1].cached_tokens == 128
    ties = 0
    for i, r in enumerate(reqs):
        ids = token_ids(r.tokens, cfg.vocab)
        ref_bf = dec_bf.forward(ids)[0]
        f_max, f_mean, f_in = chaos_floor(cfg, w, ids, ref_bf)
        e = np.abs(logits[i] - ref_bf)
        frac_in = float(np.mean(e <= ATOL + RTOL * np.abs(ref_bf)))
        print(f"req {i}: vs bf16-emulating oracle max {e.max():.4f} mean {e.mean():.5f} "
              f"in-tol {frac_in:.5f}; chaos floor max {f_max:.4f} mean {f_mean:.5f} "
              f"in-tol {f_in:.5f}")
        assert e.max() <= 1.5 * f_max and e.mean() <= 1.5 * f_mean, (e.max(), f_max, e.mean(), f_mean)
        assert frac_in >= f_in - 0.01, (frac_in, f_in)
        ref = dec.forward(ids)[0]
        err = np.abs(logits[i] - ref)
        assert err.max() <= 1.5 * FLOOR_MAX and err.mean() <= 1.5 * FLOOR_MEAN, (err.max(), err.mean())
        top = np.sort(ref_bf)[-2:]
        ties += dec_bf.check_greedy(ids, [first[i]], atol=float(f_max), rtol=0.0)
        print(f"req {i}: vs fp32 max {err.max():.4f}; top1-top2 margin {top[1] - top[0]:.4f}")
    print("near-tie exemptions:", ties)


def test_pipelined_rotations_match_sequential():
    """Async prefill + pipelined rotations (host work of r+1 under the forward of r) give the
    same cache decisions, reports and greedy tokens as the sequential loop."""
    from paper_2511_01633_b200.workload import GraphCoTWorkload

    cfg = glmx.TINY
    g = glmx.PropertyGraph.synth_powerlaw(3000, 6, seed=4, device=0)
    out = []
    for mode in ("seq", "pipe"):
        model = glmx.Model(cfg, device=0)
        kv = glmx.KvCacheState(256, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                               n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                               headroom_pages=512)
        eng = glmx.Engine(model, kv, max_requests=16, max_batch_tokens=16 * 1024, max_decode=4,
                          max_context=4096)
        ret = glmx.Retriever(g, chunk_k=8, vocab=cfg.vocab)
        wl = GraphCoTWorkload(eng, ret, n_queries=40, lanes=16, seed=5, question_pool=20,
                              node_index=glmx.NodeIndex(g))
        rows = []
        it = (wl.rotation() for _ in range(14)) if mode == "seq" else wl.rotations(14)
        for r in it:
            rows.append(([(x.cached_tokens, x.computed_tokens, x.tail_tokens) for x in r.reports],
                         r.first_tokens, r.finished))
        out.append((rows, kv.counters(), kv.snapshot_json()))
    assert out[0] == out[1]


def test_overlapped_decode_rotations_match_sequential():
    """Graph-CoT rotations with reply decode, overlapped (rotation r+1's host work under r's decode
    steps in a second thread) == the sequential rotation_with_decode loop: reports, first tokens,
    decoded counts, cache counters and snapshot."""
    from paper_2511_01633_b200.workload import GraphCoTWorkload

    cfg = glmx.TINY
    g = glmx.PropertyGraph.synth_powerlaw(3000, 6, seed=4, device=0)
    out = []
    for mode in ("seq", "overlap"):
        model = glmx.Model(cfg, device=0)
        kv = glmx.KvCacheState(256, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                               n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                               headroom_pages=512)
        eng = glmx.Engine(model, kv, max_requests=16, max_batch_tokens=16 * 1024, max_decode=8,
                          max_context=4096)
        ret = glmx.Retriever(g, chunk_k=8, vocab=cfg.vocab)
        wl = GraphCoTWorkload(eng, ret, n_queries=40, lanes=16, seed=5, question_pool=20,
                              node_index=glmx.NodeIndex(g))
        rows = []
        it = ((wl.rotation_with_decode(8) for _ in range(12)) if mode == "seq"
              else wl.rotations_with_decode(12, 8))
        for r in it:
            rows.append(([(x.cached_tokens, x.computed_tokens, x.tail_tokens) for x in r.reports],
                         r.first_tokens, r.finished, r.decoded_tokens))
        out.append((rows, kv.counters(), kv.snapshot_json()))
    assert out[0] == out[1]
    assert sum(r[3] for r in out[0][0]) > 0


@pytest.mark.parametrize("cap,policy", [(256, glmx.PRIORITY), (40, glmx.PLAIN_LRU)],
                         ids=["roomy", "self_evicting"])
def test_merged_decode_matches_separate_decode(cap, policy):
    """Continuous batching of two rotations' decode rows (decode_defer + decode_async) gives the
    same bookkeeping and the same greedy reply tokens as decoding each rotation alone -- also
    under eviction pressure, where a deferred batch's self-evicted pages must not be recycled by
    the next prefill before the merged decode has read them."""
    from paper_2511_01633_b200.workload import GraphCoTWorkload

    cfg = glmx.TINY
    g = glmx.PropertyGraph.synth_powerlaw(3000, 6, seed=4, device=0)
    out = []
    for merge in (False, True):
        model = glmx.Model(cfg, device=0)
        kv = glmx.KvCacheState(cap, 16, policy, device=0, n_layers=cfg.n_layers,
                               n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim,
                               headroom_pages=1024)
        eng = glmx.Engine(model, kv, max_requests=16, max_batch_tokens=16 * 1024, max_decode=8,
                          max_context=4096)
        ret = glmx.Retriever(g, chunk_k=8, vocab=cfg.vocab)
        wl = GraphCoTWorkload(eng, ret, n_queries=40, lanes=16, seed=5, question_pool=20,
                              node_index=glmx.NodeIndex(g))
        rows = []
        for r in wl.rotations_with_decode(11, 8, merge=merge):
            rows.append(([(x.cached_tokens, x.computed_tokens, x.tail_tokens) for x in r.reports],
                         r.first_tokens, r.finished, r.decoded_tokens))
        toks = dict(wl.decode_log)
        out.append((rows, kv.counters(), kv.snapshot_json(), toks))
        model.close()
    assert out[0][:3] == out[1][:3]
    if cap < 256:
        assert sum(out[0][1]["evictions_by_tier"]) > 0
    a, b = out[0][3], out[1][3]
    assert sorted(a) == sorted(b)
    flat_a = [t for r in sorted(a) for call in a[r] for t in call]
    flat_b = [t for r in sorted(b) for call in b[r] for t in call]
    assert len(flat_a) == len(flat_b) and len(flat_a) > 0
    # merged steps batch more rows per GEMM (other cuBLAS tiles): only fp32 near-tie flips may
    # differ; a recycled page would garble whole replies
    agree = sum(x == y for x, y in zip(flat_a, flat_b)) / len(flat_a)
    assert agree >= 0.99, agree


def test_c3_shaped_run_bookkeeping_matches_reference():
    """C3 in miniature: 96 concurrent Graph-CoT queries on a 96-block pool with four-tier
    priority eviction (pipelined rotations, RetrieveNode, K1); every prefill and set_tier replayed
    into the reference KvCacheState gives identical counters and resident snapshot."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "bench_c3.py"),
                          "--lanes", "96", "--cap", "96", "--rotations", "20", "--layers", "2",
                          "--nodes", "3000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    row = __import__("json").loads(out.stdout.strip().splitlines()[-1])
    assert row["bookkeeping_identical_to_reference"]
    assert sum(row["counters"]["evictions_by_tier"]) > 0  # the pool was under pressure


def test_reuse_off_recomputes_hits_with_same_bookkeeping():
    """Reuse on/off A/B switch (bench.py --no-reuse): with reuse off the cache hits are recomputed
    into scratch pages -- reports and cache state are the reference's, logits stay within the
    north-star tolerance of the fp32 oracle, and the cached pages are untouched (a later reuse-on
    prefill of the same prompt gives the same logits as before)."""
    model, kv, eng = make(glmx.TINY)
    dec = Decoder(glmx.TINY, model.export_all())
    p = words(90)
    warm = [glmx.Request(p, [(0, 30, 0), (30, 90, 3)], "a")]
    eng.prefill(warm)
    reqs = [glmx.Request(p[:80] + words(7, "x"), [(0, 30, 0), (30, 87, 3)], "b"),
            glmx.Request(p[:64], [(0, 64, 2)], "c")]
    _, _, on_logits = eng.prefill(reqs, want_logits=True)
    snap = kv.snapshot()
    eng.set_reuse(False)
    reps, first, off_logits = eng.prefill(reqs, want_logits=True)
    eng.set_reuse(True)
    assert [(r.cached_tokens, r.computed_tokens, r.tail_tokens) for r in reps] == [
        (80, 0, 7), (64, 0, 0)]
    assert kv.snapshot()["resident_blocks"] == snap["resident_blocks"]
    for i, r in enumerate(reqs):
        ref = dec.forward(token_ids(r.tokens, glmx.TINY.vocab))[0]
        check_logits(off_logits[i], ref)
        check_logits(on_logits[i], ref)
    _, _, again = eng.prefill(reqs, want_logits=True)
    np.testing.assert_array_equal(again, on_logits)
