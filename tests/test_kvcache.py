"""KvCacheState parity (cache.cpp) — the host block engine behind glmx_kv_* against
 (a) the reference's own golden vectors (tests/golden/golden.json, made from oracle/_ref),
 (b) the compiled reference on random op sequences (10k ops, both policies),
 (c) exhaustive small states: every cache of <= 6 blocks x every tier assignment x LRU order
     (SPEC.md:777), checked for the full eviction order,
 (d) the exact bookkeeping call sequences the reference orchestrator made in run_bench and in
     the Fig. 6 scripted run (C1) — replayed call by call.
No GPU: the kv handle is created with device = -1 (bookkeeping only)."""
import itertools
import json
import os
import random

import pytest

import oracle
import paper_2511_01633_b200 as glmx

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def report_tuple(r):
    return [r.cached_tokens, r.computed_tokens, r.tail_tokens]


def run_ops(kv, ops):
    res = []
    for toks, tiers, sess in ops:
        try:
            r = kv.prefill(toks, [tuple(t) for t in tiers], sess)
            res.append([0, report_tuple(r), [str(e) for e in r.evicted]])
        except glmx.GlmxError as e:
            res.append([e.code, [0, 0, 0], []])
    return res


def test_chain_ids_golden(golden):
    toks = [f"t{i}" for i in range(64)]
    assert [str(x) for x in glmx.chain_ids(toks, 16)] == golden["chain_ids"]
    assert hex(int(golden["chain_ids"][0])) == "0x2b241e1d1c5ffe4d"
    assert hex(int(golden["chain_ids"][3])) == "0xcf31676c1fe7074"
    assert glmx.chain_ids(toks[:15], 16) == []  # tail never hashed


def test_prefill_kats(golden):
    for kat in golden["prefill_kats"]:
        kv = glmx.KvCacheState(kat["cap"], kat["B"], kat["policy"])
        assert run_ops(kv, kat["ops"]) == kat["results"]
        c = kv.counters()
        assert [c["hits"], c["misses"]] + c["evictions_by_tier"] == kat["counters"]
        assert [[str(a), b, lu] for a, b, lu, _ in kv.resident_snapshot()] == kat["resident"]


def test_cache_exhausted_leaves_partial_state():
    kv = glmx.KvCacheState(2, 16)
    toks = [f"t{i}" for i in range(64)]
    with pytest.raises(glmx.CacheExhausted, match="need 1 evictable blocks, have 0"):
        kv.prefill(toks, [(0, 64, glmx.TIER_I)], "s")
    assert kv.resident_blocks() == 2 and kv.counters()["misses"] == 3


def test_bad_tier_map_and_config():
    kv = glmx.KvCacheState(8, 4)
    with pytest.raises(glmx.GlmxError) as e:
        kv.prefill(["a", "b"], [(0, 1, 3)], "s")
    assert e.value.code == 1
    with pytest.raises(glmx.GlmxError):
        kv.prefill(["a", "b"], [(1, 2, 3)], "s")
    with pytest.raises(glmx.ConfigError):
        glmx.KvCacheState(8, 0)


def fuzz(ref, seed, n_ops, policy):
    rnd = random.Random(seed)
    cap, B = rnd.randint(1, 12), rnd.randint(1, 5)
    rk = oracle.RefKv(ref, cap, B, policy)
    mk = glmx.KvCacheState(cap, B, policy)
    vocab = [f"w{i}" for i in range(6)]
    prefixes = [[rnd.choice(vocab) for _ in range(rnd.randint(0, 20))] for _ in range(6)]
    for op in range(n_ops):
        r = rnd.random()
        if r < 0.75:
            p = rnd.choice(prefixes) + [rnd.choice(vocab) for _ in range(rnd.randint(0, 10))]
            n = len(p)
            cuts = sorted(rnd.sample(range(n + 1), min(n + 1, rnd.randint(0, 3))))
            bounds = [0] + [c for c in cuts if 0 < c < n] + [n]
            tiers = [(bounds[i], bounds[i + 1], rnd.randint(0, 3)) for i in range(len(bounds) - 1)
                     if bounds[i] < bounds[i + 1]]
            if rnd.random() < 0.03 and tiers:  # malformed map
                tiers = tiers[1:]
            s = rnd.choice(["a", "b", "c"])
            st, rep, ev = rk.prefill(p, tiers, s)
            try:
                m = mk.prefill(p, tiers, s)
                assert st == 0, (op, st)
                assert (tuple(report_tuple(m)), m.evicted) == (rep, ev), op
            except glmx.GlmxError as e:
                assert st == e.code, (op, st, e.code)
        elif r < 0.85:
            s, f, t = rnd.choice(["a", "b", "c", ""]), rnd.randint(0, 3), rnd.randint(0, 3)
            rk.set_tier(s, f, t)
            mk.set_tier(s, f, t)
        elif r < 0.93:
            n = rnd.randint(0, 3)
            st, ids = rk.evict(n)
            try:
                assert mk.evict(n) == ids and st == 0, op
            except glmx.CacheExhausted:
                assert st == 2, op
        else:
            res = rk.resident()
            bid = rnd.getrandbits(64) if rnd.random() < 0.5 or not res else res[0][0]
            t, lu, s = rnd.randint(0, 3), rnd.randint(0, 50), rnd.choice(["a", "b", ""])
            rk.force_insert(bid, t, lu, s)
            mk.force_insert(bid, t, lu, s)
        c = mk.counters()
        assert rk.counters() == [c["hits"], c["misses"]] + c["evictions_by_tier"], op
        assert rk.resident() == [(a, b, lu) for a, b, lu, _ in mk.resident_snapshot()], op
    for bid, _, _ in rk.resident():
        assert rk.block_session(bid) == mk.block_session(bid)
    assert rk.snapshot_json() == mk.snapshot()


@pytest.mark.parametrize("policy", [glmx.PRIORITY, glmx.PLAIN_LRU])
def test_random_op_sequences_match_reference(ref, policy):
    for seed in range(40):
        fuzz(ref, seed, 250, policy)  # 10k ops per policy


@pytest.mark.parametrize("policy", [glmx.PRIORITY, glmx.PLAIN_LRU])
def test_exhaustive_small_states_eviction_order(ref, policy):
    """Every resident set of n<=6 blocks, every tier assignment, two LRU orders, full evict."""
    rnd = random.Random(policy)
    cases = 0
    for n in range(0, 7):
        for tiers in itertools.product(range(4), repeat=n):
            for order in (list(range(n)), list(reversed(range(n)))):
                rk = oracle.RefKv(ref, 16, 4, policy)
                mk = glmx.KvCacheState(16, 4, policy)
                for i in range(n):
                    bid = 1000 + i * 7919
                    lu = order[i] + (1 if rnd.random() < 0.2 else 0)  # some stamp ties -> id
                    rk.force_insert(bid, tiers[i], lu, "s")
                    mk.force_insert(bid, tiers[i], lu, "s")
                for k in range(n + 2):
                    st, ids = rk.evict(1)
                    try:
                        got = mk.evict(1)
                        assert st == 0 and got == ids
                    except glmx.CacheExhausted:
                        assert st == 2
                    if st:
                        break
                cases += 1
    assert cases == sum(2 * 4 ** n for n in range(7))


def replay_trace(trace, cap, B=16, policy=0):
    kv = glmx.KvCacheState(cap, B, policy)
    for i, op in enumerate(trace):
        if op["op"] == "set_tier":
            kv.set_tier(op["session"], op["from"], op["to"])
            continue
        tiers = [tuple(t) for t in op["tiers"]]
        if "error" in op:
            with pytest.raises(glmx.CacheExhausted):
                kv.prefill(op["tokens"], tiers, op["session"])
            return kv
        r = kv.prefill(op["tokens"], tiers, op["session"])
        assert (r.cached_tokens, r.computed_tokens, r.tail_tokens) == (
            op["cached"], op["computed"], op["tail"]), i
        assert [str(e) for e in r.evicted] == [str(e) for e in op["evicted"]], i
    return kv


def replay_segments(trace, cap, B=16, policy=0):
    """The same recorded call sequence, but each prefill fed as the PromptSegments the reference
    orchestrator tokenized (recorded inside Orchestrator::kv_prefill, oracle/rec_tokenize.hpp)
    through glmx_kv_prefill_segments -- tokenisation per segment, empty parts skipped, same-tier
    ranges merged -- instead of the already-flattened (tokens, TierMap)."""
    kv = glmx.KvCacheState(cap, B, policy)
    n = 0
    for i, op in enumerate(trace):
        if op["op"] == "set_tier":
            kv.set_tier(op["session"], op["from"], op["to"])
            continue
        segs = [(tier, text) for text, tier in op["segments"]]
        # the Python restatement (oracle.kv_prefill_inputs) is pinned to the same records
        toks, tiers = oracle.kv_prefill_inputs(segs)
        assert toks == op["tokens"] and [list(t) for t in tiers] == op["tiers"], i
        if "error" in op:
            with pytest.raises(glmx.CacheExhausted):
                kv.prefill_segments(segs, op["session"])
            return kv, n
        r = kv.prefill_segments(segs, op["session"])
        assert (r.cached_tokens, r.computed_tokens, r.tail_tokens) == (
            op["cached"], op["computed"], op["tail"]), i
        assert [str(e) for e in r.evicted] == [str(e) for e in op["evicted"]], i
        n += 1
    return kv, n


def test_recorded_prompt_segments_replay(golden):
    """a2/a3 pinned to the reference: every prefill the reference orchestrator made (Fig. 6
    scripted run and three run_bench runs, incl. eviction pressure), replayed from its segments."""
    f = golden["fig6"]
    kv, n = replay_segments(f["trace"], 4096)
    assert n == 10 and kv.snapshot() == f["kv"]
    for bt in golden["bench_traces"]:
        kv_s, n = replay_segments(bt["trace"], bt["cap"], 16, bt["policy"])
        kv_t = replay_trace(bt["trace"], bt["cap"], 16, bt["policy"])
        assert n > 0 and kv_s.resident_snapshot() == kv_t.resident_snapshot()
        assert kv_s.counters() == kv_t.counters()


def test_fig6_scripted_trace_c1(golden):
    f = golden["fig6"]
    kv = replay_trace(f["trace"], 4096)
    snap = kv.snapshot()
    assert snap == f["kv"]
    assert snap["hits"] == 22 and snap["misses"] == 12 and snap["resident_blocks"] == 12


def test_bench_traces_replay(golden):
    for bt in golden["bench_traces"]:
        kv = replay_trace(bt["trace"], bt["cap"], 16, bt["policy"])
        if bt["report"] is not None:
            assert abs(kv.hit_rate() - bt["report"]["cache_hit_rate"]) < 1e-12


def test_prefill_segments_is_orchestrator_kv_prefill(ref):
    segs = [(0, "You are   an agent.\n"), (1, ""), (1, "[Node:n1 {a:b}]\n"), (1, "x y"),
            (3, "Question: q?\nReply:\n")]
    toks, tiers = oracle.kv_prefill_inputs(segs)
    a = glmx.KvCacheState(64, 4)
    b = oracle.RefKv(ref, 64, 4, 0)
    r1 = a.prefill_segments(segs, "s")
    st, rep, _ = b.prefill(toks, tiers, "s")
    assert st == 0 and tuple(report_tuple(r1)) == rep
    assert glmx.tokenize("a\tb  c\n") == ["a", "b", "c"] == oracle.tokenize("a\tb  c\n")
