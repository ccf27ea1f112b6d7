"""K3 persistent-CTA schedule (host C++, no GPU): every key tile of every item is covered exactly
once; with many items whole items are dealt longest-first round-robin (single-query-tile items
paired two per piece); with few items each item is split into near-equal pieces (one per CTA) with
consecutive partial slots for the combine pass."""
import random

import pytest

from paper_2511_01633_b200.attention import schedule


def tiles_of(t0, ql, ctx, tpi=64):
    return (ctx - ql + min(t0 + tpi, ql) - 1) // 128 + 1


def check(reqs, n_kv=8, n_sm=148, tpi=64, pair=True):
    work = [(r, t0) for r, (ctx, ql) in enumerate(reqs) for t0 in range(0, ql, tpi)]
    ql = [q for _, q in reqs]
    ctx = [c for c, _ in reqs]
    s = schedule(work, ql, ctx, n_kv, tpi, n_sm, pair=pair)
    n_items = len(work) * n_kv
    need = [tiles_of(work[w // n_kv][1], ql[work[w // n_kv][0]], ctx[work[w // n_kv][0]], tpi)
            for w in range(n_items)]
    assert s["total_tiles"] == sum(need)
    covered = [[] for _ in range(n_items)]
    loads = []
    single = [ql[work[w // n_kv][0]] - work[w // n_kv][1] <= tpi // 2 for w in range(n_items)]
    costs = []
    for c in range(s["grid"]):
        load = 0
        for i in range(s["cta_off"][c], s["cta_off"][c + 1]):
            item, j0, j1, part = s["pieces"][i]
            assert 0 <= j0 < j1 <= need[item]
            covered[item].append((j0, j1, part))
            cost = j1 - j0
            b, b0, b1, bpart = s["partners"][i]
            if b >= 0:  # paired: two whole short single-tile items, never split
                assert pair and single[item] and single[b] and b != item
                assert need[item] <= 16 and need[b] <= 16
                assert (j0, j1, b0, b1, bpart) == (0, need[item], 0, need[b], -1)
                covered[b].append((b0, b1, bpart))
                cost = max(cost, b1 - b0)
            elif pair and single[item]:
                cost *= 0.75  # the scheduler's cost model: a lone single-tile item
            costs.append(cost)
            load += cost
        loads.append(load)
    for w in range(n_items):
        segs = sorted(covered[w])
        assert segs[0][0] == 0 and segs[-1][1] == need[w]
        assert all(a[1] == b[0] for a, b in zip(segs, segs[1:])), "gap or overlap"
        parts = [p for _, _, p in segs]
        if len(segs) == 1:
            assert parts == [-1]
        else:
            assert sorted(parts) == list(range(min(parts), min(parts) + len(parts)))
    assert s["n_partials"] <= 2 * n_sm and s["grid"] <= n_sm
    share = -(-s["total_tiles"] // s["grid"])
    if (n_items * 2 > n_sm or max(need) < 8) and not s["combine"]:  # LPT of whole items
        lens = [costs[s["cta_off"][c]] for c in range(s["grid"])]
        assert lens == sorted(lens, reverse=True)
        assert max(loads) - min(loads) <= max(need)
        assert max(loads) <= 1.3 * s["total_tiles"] / n_sm or max(need) < 16 or n_items * 2 <= n_sm
    elif n_items * 2 > n_sm:  # stream-K cut: equal ranges, edges snapped by <= share/8
        assert s["grid"] == min(n_sm, s["total_tiles"])
        assert max(loads) <= share + 2 * max(1, share // 8) + 1
    else:  # split: one piece per CTA, pieces of an item differ by <= 1 tile
        assert all(s["cta_off"][c + 1] - s["cta_off"][c] == 1 for c in range(s["grid"]))
        for w in range(n_items):
            sz = [b - a for a, b, _ in covered[w]]
            assert max(sz) - min(sz) <= 1
    comb_items = {c[0] for c in s["combine"]}
    assert comb_items == {w for w in range(n_items) if len(covered[w]) > 1}
    return s


def test_c5_batch_uses_whole_items():
    s = check([(8192 + 128, 128)] * 8)  # 128 items of 65 tiles on 148 SMs
    assert s["grid"] == 128 and not s["combine"]


def test_long_tail_falls_back_to_stream_k():
    # 7 requests x 3 query blocks x 8 kv heads = 168 items of ~257 tiles on 148 SMs: LPT would
    # need two waves; the stream-K cut balances the tiles
    s = check([(32768 + 134, 134)] * 7, pair=False)
    assert s["grid"] == 148 and s["combine"] and s["n_partials"] <= 2 * 148
    # the 56 six-token blocks have ~257 key tiles each: too long to pair (two K/V streams per CTA
    # would exceed the L2 throughput), so the paired schedule is the same stream-K cut
    s = check([(32768 + 134, 134)] * 7)
    assert s["grid"] == 148 and s["combine"]
    assert all(b == -1 for b, _, _, _ in s["partners"])


def test_single_long_query_is_split_across_sms():
    s = check([(32768 + 100, 100)])  # 16 items -> 9 pieces each
    assert s["grid"] == 144 and len(s["combine"]) == 16 and s["n_partials"] == 144


def test_short_items_are_never_split():
    s = check([(200, 40)] * 64)
    assert not s["combine"]


def test_ragged_random_batches():
    rnd = random.Random(0)
    for trial in range(30):
        reqs = []
        for _ in range(rnd.randrange(1, 70)):
            ql = rnd.randrange(1, 400)
            reqs.append((ql + rnd.choice([0, rnd.randrange(0, 5000)]), ql))
        check(reqs, n_kv=rnd.choice([8, 4]), n_sm=rnd.choice([148, 7, 1]), pair=trial % 3 != 0)


def test_fewer_tiles_than_sms():
    s = check([(1, 1)])  # 8 single-tile items: one CTA each beats pairing
    assert s["grid"] == 8 and len(s["pieces"]) == 8
    assert all(b == -1 for b, _, _, _ in s["partners"])


def test_short_items_are_not_split_even_when_few():
    s = check([(300, 1)] * 8)  # decode step: 64 items of 3 key tiles
    assert not s["combine"] and s["grid"] == 64


def test_many_single_tile_items_are_paired():
    s = check([(300, 1)] * 37)  # 296 items: two waves alone, one wave of pairs
    assert s["grid"] == 148 and all(b >= 0 for b, _, _, _ in s["partners"])
    s = check([(300, 1)] * 37, pair=False)
    assert s["grid"] == 148 and len(s["pieces"]) == 296


def test_pairs_match_lengths():
    # 16 single-tile items of 1..16 key tiles: pairs are neighbours in length order
    reqs = [(128 * k, 20) for k in range(1, 17)]
    s = check(reqs, n_kv=1, n_sm=4)
    assert s["grid"] == 4
    for (a, _, a1, _), (b, _, b1, _) in zip(s["pieces"], s["partners"]):
        assert b >= 0 and abs(a1 - b1) <= 1


def test_two_tile_items_are_not_paired():
    s = check([(5000, 64)] * 4 + [(3000, 20)] * 3)
    for (a, _, _, _), (b, _, _, _) in zip(s["pieces"], s["partners"]):
        if a < 32:
            assert b == -1


@pytest.mark.parametrize("n_sm", [1, 2, 148])
def test_single_long_item(n_sm):
    check([(32768, 1)], n_kv=1, n_sm=n_sm)


def test_pairing_boundaries():
    # a block of 32 tokens (= tokens_per_item / 2) uses one query tile and may pair; 33 tokens
    # need two tiles and never pair; single-tile items longer than 16 key tiles never pair
    reqs = [(100, 32)] * 300  # 2400 single-tile items of 1 key tile: two waves alone
    s = check(reqs)
    assert any(b >= 0 for b, _, _, _ in s["partners"])
    s = check([(100, 33)] * 300)
    assert all(b == -1 for b, _, _, _ in s["partners"])
    s = check([(128 * 17, 32)] * 40)  # 17 key tiles each
    assert all(b == -1 for b, _, _, _ in s["partners"])
    s = check([(128 * 16, 32)] * 40)  # 16 key tiles each: pairable
    assert s["grid"] <= 148
