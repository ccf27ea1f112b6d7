"""K2 (fused RoPE + paged KV append) against a plain PyTorch fp32 reference through the C-ABI
hook glmx_rope_kv_append_run: V pages byte-exact, RoPE'd Q/K within one bf16 rounding of the fp32
rotation (the kernel rotates in fp32 and rounds once), untouched pages unchanged."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T", [1, 7, 64, 767, 768, 1000, 2501])  # ragged CTA tails (3 tokens per CTA) and the old 768-token crossover
def test_append_matches_reference(T):
    check_append(T, 32, 8)


# head counts whose 4-head passes do not fill the 3-pass warp groups evenly: C1's tiny decoder
# (4 q / 2 kv: 2 passes, one partial group), 20 heads (5 passes: 3 + 2), MHA 8/8 (6 passes)
@pytest.mark.parametrize("H,Hkv", [(4, 2), (12, 4), (8, 8)])
@pytest.mark.parametrize("T", [1, 5, 301])
def test_append_head_configs(T, H, Hkv):
    check_append(T, H, Hkv)


def check_append(T, H, Hkv):
    from paper_2511_01633_b200.ops import rope_kv_append
    from torch_refs import reference_rope

    hd, B, L, layer = 128, 16, 3, 2
    g = torch.Generator().manual_seed(T)
    n_pages = (T + B - 1) // B + 5
    qkv = torch.randn((T, (H + 2 * Hkv) * hd), generator=g).to(torch.bfloat16).cuda()
    pos = torch.randint(0, 32768, (T,), generator=g, dtype=torch.int32).cuda()
    perm = torch.randperm(n_pages, generator=g)[: (T + B - 1) // B]
    slot = torch.tensor([int(perm[t // B]) * B + t % B for t in range(T)], dtype=torch.int64).cuda()
    pool = torch.randn((n_pages, L, 2, Hkv, B, hd), generator=g).to(torch.bfloat16).cuda()
    before = pool.clone()
    q_out = torch.empty((T, H, hd), dtype=torch.bfloat16, device="cuda")
    rope_kv_append(qkv, pos, slot, pool, q_out, H, Hkv, layer=layer)
    torch.cuda.synchronize()
    x = qkv.view(T, H + 2 * Hkv, hd)
    q_ref = reference_rope(x[:, :H], pos)
    k_ref = reference_rope(x[:, H:H + Hkv], pos)
    v_ref = x[:, H + Hkv:]
    tol = lambda ref: 2.0 ** -8 * ref.abs() + 1e-6  # noqa: E731  one bf16 rounding
    assert ((q_out.float() - q_ref).abs() <= tol(q_ref)).all()
    page, off = (slot // B).long(), (slot % B).long()
    k_got = pool[page, layer, 0, :, off]  # [T][Hkv][hd]
    v_got = pool[page, layer, 1, :, off]
    assert ((k_got.float() - k_ref).abs() <= tol(k_ref)).all()
    assert torch.equal(v_got, v_ref)
    # nothing else written: other layers, and rows not addressed by a slot
    mask = torch.ones_like(pool, dtype=torch.bool)
    mask[page, layer, :, :, off] = False
    assert torch.equal(pool[mask], before[mask])


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "scalar"])
@pytest.mark.parametrize("n", [1, 37, 1000])
def test_kv_gather_matches_reference(impl, n):
    from paper_2511_01633_b200.ops import kv_gather

    Hkv, hd, B, L = 8, 128, 16, 3
    g = torch.Generator().manual_seed(n)
    pool = torch.randn((n + 13, L, 2, Hkv, B, hd), generator=g).to(torch.bfloat16).cuda()
    pages = torch.randperm(n + 13, generator=g)[:n].tolist()
    for layer, kv in ((0, 0), (2, 1)):
        out = torch.full((n * B, Hkv, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
        kv_gather(pool, pages, layer, kv, out, impl=impl)
        torch.cuda.synchronize()
        want = pool[torch.tensor(pages, device="cuda"), layer, kv].permute(0, 2, 1, 3).reshape(n * B, Hkv, hd)
        assert torch.equal(out, want)
