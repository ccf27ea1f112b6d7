"""TEST INFRASTRUCTURE ONLY — numpy fp32 Llama-style decoder (the tensor-math oracle).

PARITY UNPINNED BY THE REFERENCE: the reference has no transformer ("real transformer
KV tensors (replaced by a token-block cost simulator)").  This restatement is
builder-authored and follows standard Llama-3 semantics:
  RMSNorm eps 1e-5 (weight multiply after normalisation), RoPE theta 500000 rotate-half on the
  post-projection Q/K with absolute positions, GQA (H/Hkv query heads share a kv head), causal
  mask, SwiGLU (silu(gate) * up), untied lm_head, greedy = first argmax.
It is pinned to the reference only through the token/block layout: positions are indices in the
concatenated per-segment TokenSeq (orchestrator.cpp:81-97); token ids are fnv1a(bytes) mod V.
Weights are the engine's own bf16 weights (exported), promoted to fp32; activations stay fp32.
"""
from __future__ import annotations

import numpy as np


def fnv1a(b: bytes, h: int = 14695981039346656037) -> int:
    for c in b:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def token_ids(tokens, vocab):
    return [fnv1a(t.encode() if isinstance(t, str) else t) % vocab for t in tokens]


def inv_freq(head_dim, theta):
    i = np.arange(0, head_dim // 2, dtype=np.float64)
    return (1.0 / np.power(float(np.float32(theta)), 2.0 * i / head_dim)).astype(np.float32)


def rope(x, pos, inv):
    """x [n, h, hd] fp32; rotate-half with fp32 angles pos*inv."""
    ang = (pos.astype(np.float32)[:, None] * inv[None, :]).astype(np.float32)
    cos = np.cos(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    sin = np.sin(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    return np.concatenate([a * cos - b * sin, b * cos + a * sin], axis=-1)


def rmsnorm(x, w, eps):
    var = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True)
    return (x / np.sqrt(var + eps)) * w


def bf16_round(x):
    """Round fp32 -> bf16 (round-to-nearest-even) -> fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


class Decoder:
    SITES = ("h1", "qkv", "q", "k", "v", "P", "attn", "h2", "gu", "act", "hf")

    def __init__(self, cfg, weights, emulate_bf16=False):
        """emulate_bf16: diagnostic mode that rounds activations to bf16 at the given sites
        (True = all of SITES); the parity oracle is the fp32 default (no rounding)."""
        self.c = cfg
        self.w = weights
        self.inv = inv_freq(cfg.head_dim, cfg.rope_theta)
        sites = set(self.SITES) if emulate_bf16 is True else set(emulate_bf16 or ())
        self.r = lambda a, site: bf16_round(a) if site in sites else a
        # with P emulated, the softmax follows the engine's K3 algorithm (attn_tc.cu): 128-key
        # tiles, base-2 exponent with a lazily raised reference max (only when a tile's row max
        # exceeds it by > 2^8), P rounded to bf16 for PV while the row sum adds the fp32 P
        self.lazy_p = "P" in sites

    def _attn_tiled(self, q, k, v, mask):
        """One head: q [n, hd], k / v [m, hd], mask [n, m] -> [n, hd] (fp32)."""
        n, hd = q.shape
        scale = np.float32(1.0 / np.sqrt(hd) * 1.4426950408889634)
        s_all = (q @ k.T).astype(np.float32)
        m_used = np.full(n, -np.inf, dtype=np.float32)
        l = np.zeros(n, dtype=np.float32)
        o = np.zeros((n, v.shape[1]), dtype=np.float32)
        for j0 in range(0, k.shape[0], 128):
            s = np.where(mask[:, j0:j0 + 128], s_all[:, j0:j0 + 128], -np.inf).astype(np.float32)
            mx = s.max(axis=1) * scale
            grow = mx > m_used + np.float32(8.0)
            with np.errstate(invalid="ignore", over="ignore"):
                alpha = np.where(grow, np.exp2(m_used - mx), np.float32(1.0)).astype(np.float32)
            alpha = np.where(np.isnan(alpha), np.float32(0.0), alpha)
            m_used = np.where(grow, mx, m_used)
            neg_m = np.where(np.isinf(m_used), np.float32(0.0), -m_used).astype(np.float32)
            p = np.exp2(s * scale + neg_m[:, None]).astype(np.float32)
            l = l * alpha + p.sum(axis=1, dtype=np.float32)
            o = o * alpha[:, None] + bf16_round(p) @ v[j0:j0 + 128]
        return o / l[:, None]

    def forward(self, ids, pos=None, past=None, return_all=False):
        """ids [n]; past: per-layer (K [p,Hkv,hd], V) of preceding positions.  Returns logits of
        the last position (or all) and the updated cache."""
        c, w = self.c, self.w
        n = len(ids)
        p0 = 0 if past is None else past[0][0].shape[0]
        if pos is None:
            pos = np.arange(p0, p0 + n)
        H, Hkv, hd = c.n_heads, c.n_kv_heads, c.head_dim
        G = H // Hkv
        r = self.r
        x = w["embed"][np.asarray(ids)].astype(np.float32)
        new_past = []
        for l, lw in enumerate(w["layers"]):
            h = r(rmsnorm(x, lw["attn_norm"], c.norm_eps), "h1")
            qkv = r(h @ lw["wqkv"].T, "qkv")
            q = qkv[:, :H * hd].reshape(n, H, hd)
            k = qkv[:, H * hd:(H + Hkv) * hd].reshape(n, Hkv, hd)
            v = qkv[:, (H + Hkv) * hd:].reshape(n, Hkv, hd)
            q = r(rope(q, pos, self.inv), "q")
            k = r(rope(k, pos, self.inv), "k")
            v = r(v, "v")
            if past is not None:
                k = np.concatenate([past[l][0], k], axis=0)
                v = np.concatenate([past[l][1], v], axis=0)
            new_past.append((k, v))
            m = k.shape[0]
            out = np.empty((n, H, hd), dtype=np.float32)
            kpos = np.arange(m)
            mask = kpos[None, :] <= np.asarray(pos)[:, None]
            for hh in range(H):
                kh = hh // G
                if self.lazy_p:
                    out[:, hh, :] = self._attn_tiled(q[:, hh, :], k[:, kh, :], v[:, kh, :], mask)
                    continue
                s = (q[:, hh, :] @ k[:, kh, :].T) / np.sqrt(hd)
                s = np.where(mask, s, -np.inf)
                s = s - s.max(axis=1, keepdims=True)
                pr = np.exp(s)
                den = pr.sum(axis=1, keepdims=True)
                out[:, hh, :] = (r(pr, "P") @ v[:, kh, :]) / den
            x = x + r(out.reshape(n, H * hd), "attn") @ lw["wo"].T
            h = r(rmsnorm(x, lw["mlp_norm"], c.norm_eps), "h2")
            gu = r(h @ lw["w_gate_up"].T, "gu")
            g, u = gu[:, :c.d_ff], gu[:, c.d_ff:]
            act = r(g / (1.0 + np.exp(-g)) * u, "act")
            x = x + act @ lw["w_down"].T
        rows = x if return_all else x[-1:]
        hf = r(rmsnorm(rows, w["final_norm"], c.norm_eps), "hf")
        logits = hf @ w["lm_head"].T
        return (logits if return_all else logits[0]), new_past

    def greedy(self, ids, steps):
        logits, past = self.forward(ids)
        out = []
        tok = int(np.argmax(logits))
        out.append(tok)
        for _ in range(steps):
            logits, past = self.forward([tok], past=past)
            tok = int(np.argmax(logits))
            out.append(tok)
        return out  # out[0] = prefill's first token, then `steps` decode tokens

    def check_greedy(self, ids, got, atol=2e-2, rtol=1e-2):
        """Teacher-forced greedy check of a GPU token sequence got = [first, d1, d2, ...]:
        every token must be the oracle's first argmax, unless the oracle's top-1/top-2 margin is
        within the bf16-vs-fp32 tolerance (a near-tie), in which case the GPU's pick must be one
        of the tied candidates.  Returns the number of near-tie steps."""
        logits, past = self.forward(ids)
        ties = 0
        for i, tok in enumerate(got):
            best = int(np.argmax(logits))
            if tok != best:
                tol = 2 * (atol + rtol * abs(float(logits[best])))
                assert float(logits[best]) - float(logits[tok]) <= tol, (
                    f"step {i}: gpu {tok} ({logits[tok]:.5f}) vs oracle {best} ({logits[best]:.5f})")
                ties += 1
            if i + 1 < len(got):
                logits, past = self.forward([tok], past=past)
        return ties
