"""K3 (paged causal GQA prefill attention) against a plain PyTorch fp32 reference, through the
C-ABI kernel hook glmx_attention_run.  Tolerance from the north star: bf16 output vs fp32 within
max-abs 2e-2 and rel 1e-2 (|err| <= 2e-2 + 1e-2 * |ref|)."""
import random

import pytest

torch = pytest.importorskip("torch")

from torch_refs import reference_attention

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 1e-2


def _case(reqs, L=2, Hkv=8, G=4, hd=128, B=16, layer=1, seed=0, extra_pages=7):
    """reqs: list of (ctx_len, q_len).  Pages are handed out in a shuffled order so block
    tables are non-contiguous; rows of different requests are packed back to back."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    n_pages = sum((c + B - 1) // B for c, _ in reqs) + extra_pages
    pool = torch.randn((n_pages, L, 2, Hkv, B, hd), generator=g).to(torch.bfloat16).cuda()
    rows = sum(q for _, q in reqs)
    q = torch.randn((rows, Hkv * G, hd), generator=g).to(torch.bfloat16).cuda()
    perm = list(range(n_pages))
    random.Random(seed).shuffle(perm)
    bt, qs, ql, ctx = [], [], [], []
    p = r = 0
    for c, n in reqs:
        k = (c + B - 1) // B
        bt.append(perm[p:p + k])
        p += k
        qs.append(r)
        ql.append(n)
        ctx.append(c)
        r += n
    return q, pool, qs, ql, ctx, bt, layer


def _check(impl, reqs, **kw):
    import paper_2511_01633_b200.attention as A

    q, pool, qs, ql, ctx, bt, layer = _case(reqs, **kw)
    o = torch.full_like(q, float("nan"))
    A.paged_attention(q, o, pool, qs, ql, ctx, bt, layer=layer, impl=impl)
    torch.cuda.synchronize()
    ref = reference_attention(q, pool, qs, ql, ctx, bt, layer=layer)
    err = (o.float() - ref).abs()
    bound = ATOL + RTOL * ref.abs()
    assert torch.isfinite(o.float()).all(), "unwritten or non-finite output rows"
    bad = (err > bound).sum().item()
    assert bad == 0, f"{bad} elements out of tolerance, max err {err.max().item():.4g}"
    return err.max().item()


MIXED = [(1, 1), (16, 16), (37, 37), (200, 5), (300, 33), (129, 64), (1000, 130), (70, 65),
         (2050, 1), (513, 97)]


def test_mixed_requests():
    _check(0, MIXED)


def test_long_prefix_short_suffix():
    # C5 shape: long cached prefix, ~100-token suffix
    _check(0, [(4096 + 100, 100), (8200, 120), (3000, 64)], seed=1)


def test_full_causal_prefill():
    # cold prompt: every key computed in this batch (diagonal tiles everywhere)
    _check(0, [(1100, 1100), (64, 64), (65, 65)], seed=2)


def test_many_items_more_than_sms():
    # > 148 work items: the persistent CTAs walk several items each (pipeline across items)
    reqs = [(random.Random(i).randrange(40, 900), 0) for i in range(40)]
    reqs = [(c, max(1, min(c, random.Random(100 + i).randrange(1, 200)))) for i, (c, _) in
            enumerate(reqs)]
    _check(0, reqs, seed=3)


def test_gqa_8_heads_per_kv_head():
    _check(0, [(500, 77), (40, 40)], Hkv=4, G=8, seed=4)


def test_layer_offset_and_single_layer_pool():
    _check(0, [(333, 33)], L=1, layer=0, seed=5)


def test_single_long_query_split_and_combined():
    # 16 items < 148 / 2: every item's key range is split over ~9 CTAs, partials merged
    _check(0, [(6000 + 100, 100)], seed=6)
    _check(0, [(3000, 1)], seed=7)  # decode-like: one row, 8 items


# Split pieces that start past some rows' positions (few items: every item's key range is cut
# into ~148 / items pieces).  ctx = 2060, q = 20: the piece of key tile 16 (keys 2048..2059) holds
# no visible key for the rows at positions 2040..2047, whose partial must be (m=-inf, l=0, O=0),
# not NaN, and must drop out of the combine.
SPLIT_EDGE = [(c, q) for c in (900, 1025, 1064, 1500, 2049, 2060, 2100, 2400)
              for q in (1, 8, 20, 33, 64)]


@pytest.mark.parametrize("ctx,ql", SPLIT_EDGE, ids=[f"{c}x{q}" for c, q in SPLIT_EDGE])
def test_split_pieces_with_invisible_rows(ctx, ql):
    _check(0, [(ctx, ql)], seed=ctx * 100 + ql)


def test_split_pieces_few_requests_unaligned():
    # 3 and 9 requests (24 / 72 items <= 74): still the split path, several items per request
    _check(0, [(2060, 20), (1064, 64), (1300, 37)], seed=31)
    _check(0, [(1000 + 131 * i, 5 + 7 * i) for i in range(9)], seed=32)


def test_split_schedule_reaches_invisible_rows():
    """The schedule really produces a piece whose first key lies past some rows (the case the
    tests above must cover): item rows at 2040..2059, a piece starting at key 2048."""
    import paper_2511_01633_b200.attention as A

    sc = A.schedule([(0, 0)], [20], [2060], n_kv_heads=8, tokens_per_item=64)
    starts = {j0 for _, j0, _, _ in sc["pieces"]}
    assert 16 in starts and sc["combine"], sc["pieces"][:20]


def test_stream_k_cut_unaligned_rows():
    # 21 requests x 8 kv heads = 168 long items on 148 SMs: the LPT makespan has a long tail, so
    # the flattened tile sequence is cut into equal ranges (stream-K) with partials + combine
    import paper_2511_01633_b200.attention as A

    reqs = [(2060 + 37 * i, 40 + (i % 5)) for i in range(21)]
    sc = A.schedule([(i, 0) for i in range(21)], [q for _, q in reqs], [c for c, _ in reqs],
                    n_kv_heads=8, tokens_per_item=64)
    assert sc["combine"] and sc["grid"] == 148  # the stream-K path, with split items
    _check(0, reqs, seed=33)


def test_paired_single_tile_items():
    # > 148 single-query-tile blocks (<= 32 tokens each): the schedule pairs them two per CTA
    # pass (one per softmax warpgroup, separate K/V streams of different lengths)
    rnd = random.Random(8)
    reqs = []
    for _ in range(48):
        ql = rnd.randrange(1, 33)
        reqs.append((ql + rnd.choice([0, rnd.randrange(0, 3000)]), ql))
    _check(0, reqs, seed=8)


def test_paired_items_mixed_with_two_tile_items():
    rnd = random.Random(9)
    reqs = [(rnd.randrange(100, 2500), 0) for _ in range(40)]
    reqs = [(c, min(c, rnd.choice([1, 7, 32, 33, 64, 96, 150]))) for c, _ in reqs]
    _check(0, reqs, seed=9)


@pytest.mark.parametrize("n_req", [1, 8, 64, 200])
def test_decode_kernel_one_token_rows(n_req):
    # K3d (CUDA-core flash-decoding, impl 2): one query token per request, contexts from a single
    # key to several thousand (one split per item for large batches, many for small ones)
    rnd = random.Random(n_req)
    reqs = [(rnd.choice([1, 15, 16, 17, 31, rnd.randrange(2, 400), rnd.randrange(400, 4000)]), 1)
            for _ in range(n_req)]
    _check(2, reqs, seed=10 + n_req)


def test_decode_kernel_matches_tc_kernel():
    import paper_2511_01633_b200.attention as A

    reqs = [(c, 1) for c in (5, 100, 333, 1024, 2049)]
    q, pool, qs, ql, ctx, bt, layer = _case(reqs, seed=21)
    o2 = torch.empty_like(q)
    o0 = torch.empty_like(q)
    A.paged_attention(q, o2, pool, qs, ql, ctx, bt, layer=layer, impl=2)
    A.paged_attention(q, o0, pool, qs, ql, ctx, bt, layer=layer, impl=0)
    torch.cuda.synchronize()
    assert (o2.float() - o0.float()).abs().max().item() < 2e-2
