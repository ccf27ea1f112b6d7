"""Plain PyTorch fp32 restatements of the K2 / K3 kernels, used only as the numerics checkers of
the GPU tests (the product package never imports this module)."""


def reference_attention(q, pool, q_start, q_len, ctx_len, block_table, layer=0):
    """Plain PyTorch fp32 restatement (causal GQA over absolute positions) for the tests."""
    import torch

    n_pages, L, _, Hkv, B, hd = pool.shape
    H = q.shape[1]
    G = H // Hkv
    out = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    scale = hd ** -0.5
    for r in range(len(q_len)):
        ctx, ql, qs = int(ctx_len[r]), int(q_len[r]), int(q_start[r])
        pages = torch.tensor(block_table[r][:(ctx + B - 1) // B], device=pool.device,
                             dtype=torch.long)
        k = pool[pages, layer, 0].float().permute(1, 0, 2, 3).reshape(Hkv, -1, hd)[:, :ctx]
        v = pool[pages, layer, 1].float().permute(1, 0, 2, 3).reshape(Hkv, -1, hd)[:, :ctx]
        qq = q[qs:qs + ql].float().permute(1, 0, 2)                     # [H][ql][hd]
        kk = k.repeat_interleave(G, dim=0)                               # [H][ctx][hd]
        vv = v.repeat_interleave(G, dim=0)
        s = torch.matmul(qq, kk.transpose(1, 2)) * scale                 # [H][ql][ctx]
        pos = torch.arange(ctx - ql, ctx, device=q.device)[:, None]
        key = torch.arange(ctx, device=q.device)[None, :]
        s = s.masked_fill(key > pos, float("-inf"))
        out[qs:qs + ql] = torch.matmul(torch.softmax(s, dim=-1), vv).permute(1, 0, 2)
    return out


def reference_rope(x, pos, rope_theta=500000.0):
    """fp32 rotate-half RoPE, angles as in oracle/decoder.py:rope (fp32 pos * fp32 inv_freq, then
    cos/sin in fp64): x [T][heads][hd]."""
    import torch

    hd = x.shape[-1]
    inv = (1.0 / (float(torch.tensor(rope_theta, dtype=torch.float32)) **
                  (torch.arange(0, hd // 2, dtype=torch.float64) * 2.0 / hd))).float()
    ang = (pos.cpu().float()[:, None] * inv[None, :]).double()
    cos = torch.cos(ang).float().to(x.device)[:, None, :]
    sin = torch.sin(ang).float().to(x.device)[:, None, :]
    a, b = x[..., :hd // 2].float(), x[..., hd // 2:].float()
    return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)
