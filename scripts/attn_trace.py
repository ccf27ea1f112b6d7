"""K3 pipeline timeline of CTA 0 (trace build): per key tile, clock64 stamps of the MMA warp and
both softmax warpgroups; prints the steady-state phase durations in SM cycles.

  GLMX_LIB=paper_2511_01633_b200/libglmx_trace.so python scripts/attn_trace.py [P] [batch]"""
import ctypes as C
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GLMX_LIB", os.path.join(ROOT, "paper_2511_01633_b200", "libglmx_trace.so"))

import torch  # noqa: E402

import paper_2511_01633_b200.attention as A  # noqa: E402
from paper_2511_01633_b200._lib import lib  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
s = int(sys.argv[3]) if len(sys.argv) > 3 else 128
H, Hkv, hd, B = 32, 8, 128, 16
ctx = P + s
pp = (ctx + B - 1) // B
pool = torch.randn((nb * pp, 1, 2, Hkv, B, hd), device="cuda").to(torch.bfloat16)
q = torch.randn((nb * s, H, hd), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
perm = list(range(nb * pp))
random.Random(0).shuffle(perm)
bt = [perm[i * pp:(i + 1) * pp] for i in range(nb)]
args = (q, o, pool, [i * s for i in range(nb)], [s] * nb, [ctx] * nb, bt)
if os.environ.get("GLMX_TRACE_SHAPES"):  # "file.json:index": one ragged batch [[ctx, q_len], ...]
    import json
    fn, idx = os.environ["GLMX_TRACE_SHAPES"].rsplit(":", 1)
    reqs = json.load(open(fn))[int(idx)]
    pages = [(c + B - 1) // B for c, _ in reqs]
    pool = torch.randn((sum(pages), 1, 2, Hkv, B, hd), device="cuda").to(torch.bfloat16)
    rows = sum(n for _, n in reqs)
    q = torch.randn((rows, H, hd), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    perm = list(range(sum(pages)))
    random.Random(0).shuffle(perm)
    bt, qs, p0, r0 = [], [], 0, 0
    for (c, n), k in zip(reqs, pages):
        bt.append(perm[p0:p0 + k])
        qs.append(r0)
        p0 += k
        r0 += n
    args = (q, o, pool, qs, [n for _, n in reqs], [c for c, _ in reqs], bt)
A.paged_attention(*args, reps=2)
buf = (C.c_int64 * (16 * 1024))()
lib().glmx_attn_trace_read(buf, 16 * 1024)  # clear
ms = A.paged_attention(*args, reps=1)
n = lib().glmx_attn_trace_read(buf, 16 * 1024)
assert n > 0, "not a trace build"
ev = [[buf[e * 1024 + j] for j in range(1024)] for e in range(16)]
n_t = max(j for j in range(1024) if ev[6][j]) + 1
if "--raw" in sys.argv:  # per-tile absolute timeline (cycles from the first stamp)
    t0 = min(x for e in ev for x in e[:n_t] if x)
    for j in range(n_t):
        print(j, " ".join(f"{(ev[e][j] - t0) if ev[e][j] else -1:7d}" for e in range(16)))
cta = [buf[15 * 1024 + 1023 - k] for k in range(3)]
if all(cta):
    first_k = ev[14][0] if ev[14][0] else cta[1]
    print(f"CTA 0: setup (barrier init + TMEM alloc) {cta[1] - cta[0]} cyc, setup -> first K issue "
          f"{first_k - cta[1]} cyc, first K issue -> first S ready {ev[6][0] - first_k} cyc, "
          f"last P -> teardown {cta[2] - max(ev[7][n_t - 1], ev[10][n_t - 1])} cyc, total {cta[2] - cta[0]} cyc")
names = {"mma: wait P0": (0, 1), "mma: issue PV0+S0": (1, 2), "mma: wait P1": (2, 3),
         "mma: issue PV1+S1": (3, 4), "WG0: wait S0": (5, 6), "WG0: softmax": (6, 7),
         "WG1: wait S1": (8, 9), "WG1: softmax": (9, 10)}
lo, hi = (4, n_t - 4) if n_t > 12 else (0, n_t - 1)
print(f"P={P} batch={nb}: kernel {ms * 1e3:.1f} us, CTA0 tiles {n_t}")
for k, (a, b) in names.items():
    d = [ev[b][j] - ev[a][j] for j in range(lo, hi)]
    print(f"  {k:22s} mean {sum(d) / len(d):8.1f} cyc  min {min(d):7d}  max {max(d):7d}")
per = [ev[6][j + 1] - ev[6][j] for j in range(lo, hi - 1)]
print(f"  {'period (WG0 S ready)':22s} mean {sum(per) / len(per):8.1f} cyc")
lat = [ev[6][j + 1] - ev[7][j] for j in range(lo, hi - 1)]
print(f"  {'WG0 P arrive -> next S':22s} mean {sum(lat) / len(lat):8.1f} cyc")
lat = [ev[1][j] - ev[7][j] for j in range(lo, hi)]
print(f"  {'WG0 P arrive -> MMA sees':22s} mean {sum(lat) / len(lat):8.1f} cyc")
d = [ev[11][j] - ev[1][j] for j in range(lo, hi)]
print(f"  {'mma: V_j wait':22s} mean {sum(d) / len(d):8.1f} cyc")
d = [ev[13][j] - ev[12][j] for j in range(lo, hi)]
print(f"  {'mma: K_j+1 wait':22s} mean {sum(d) / len(d):8.1f} cyc")
d = [ev[13][j] - ev[14][j + 1] for j in range(lo, hi)]
print(f"  {'K_j+1 issue->consumed':22s} mean {sum(d) / len(d):8.1f} cyc")
d = [ev[11][j] - ev[15][j] for j in range(lo, hi)]
print(f"  {'V_j issue->consumed':22s} mean {sum(d) / len(d):8.1f} cyc")
print("  tensor work per tile: 4 x 128x128x128 MMAs = 2048 cyc at 8192 flop/clk")
