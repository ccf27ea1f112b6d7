"""The priority-vs-LRU adversarial workload (the reference ships none):
retrieved-chunk notebooks (tier II) re-read every round between floods of one-off tier-IV agent
prompts.  Four-tier priority eviction keeps the notebooks and beats plain LRU by a wide margin;
for both policies every report and eviction equals the reference's KvCacheState."""
import pytest

import oracle
import paper_2511_01633_b200 as glmx
from oracle import kv_prefill_inputs
from paper_2511_01633_b200.workload import adversarial_priority_ops


def run(policy, ops, cap, ref):
    ours = glmx.KvCacheState(cap, 16, policy, device=-1)
    rk = oracle.RefKv(ref, cap, 16, policy)
    hot_hit = hot_tok = 0
    for _, segs, sess in ops:
        toks, tiers = kv_prefill_inputs(segs)
        st, rep, ev = rk.prefill(toks, tiers, sess)
        r = ours.prefill_segments(segs, sess)
        assert st == 0
        assert ((r.cached_tokens, r.computed_tokens, r.tail_tokens), list(r.evicted)) == (rep, ev)
        if sess.startswith("hot"):
            hot_hit += r.cached_tokens
            hot_tok += len(toks)
    assert ours.snapshot() == rk.snapshot_json()
    return ours.hit_rate(), hot_hit / hot_tok


def test_priority_beats_lru_on_the_adversarial_stream(ref):
    ops = adversarial_priority_ops(n_hot=8, rounds=10, n_cold=24)
    pri, pri_hot = run(glmx.PRIORITY, ops, 256, ref)
    lru, lru_hot = run(glmx.PLAIN_LRU, ops, 256, ref)
    # hot reasoning prompts: priority keeps the tier-II notebooks resident across floods
    assert pri_hot > 0.8 and lru_hot < 0.3, (pri_hot, lru_hot)
    assert pri > lru


@pytest.mark.parametrize("cap", [128, 512])
def test_adversarial_stream_parity_other_capacities(ref, cap):
    ops = adversarial_priority_ops(n_hot=6, rounds=4, n_cold=16, seed=cap)
    for policy in (glmx.PRIORITY, glmx.PLAIN_LRU):
        run(policy, ops, cap, ref)
