"""torchrun --nproc-per-node 2: the pipelined epoch protocol for cross-GPU prefix hits
(PeerExchange.before_bookkeeping / after_wait, GraphCoTWorkload.rotations(peer=...)) against the
sequential one (epoch_begin / epoch_end around every rotation), both ranks on one GPU (one per GPU
in production).  A small pool forces evictions, so pages named in a published directory are
evicted (and deferred) while peers may still copy them.  Checks:
  * cache counters per rank identical (the directory only turns misses into copies),
  * peer hits happen in both protocols,
  * the greedy first tokens agree (a page recycled while a peer still copies it would feed
    garbage KV into the peer's attention),
  * the pool never runs out (deferred pages are released with the one-rotation lag).
Prints "peer_pipeline_check ok" on success."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.sharding import PeerExchange  # noqa: E402
from paper_2511_01633_b200.workload import GraphCoTWorkload  # noqa: E402

ROT = int(os.environ.get("GLMX_CHECK_ROTATIONS", "14"))
CAP = int(os.environ.get("GLMX_CHECK_CAPACITY", "224"))  # blocks per rank: forces evictions
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("GLMX_PEER_DEVICE", "0"))
torch.cuda.set_device(dev)
cfg = glmx.TINY
g = glmx.PropertyGraph.synth_powerlaw(3000, 8, seed=1, device=dev)
ret = glmx.Retriever(g, chunk_k=16, vocab=cfg.vocab)
model = glmx.Model(cfg, dev)


def run(pipelined, decode=False):
    kv = glmx.KvCacheState(CAP, 16, glmx.PRIORITY, device=dev, n_layers=cfg.n_layers,
                           n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, headroom_pages=1024)
    eng = glmx.Engine(model, kv, max_requests=16, max_batch_tokens=16 * 1024, max_decode=4,
                      max_context=4096)
    wl = GraphCoTWorkload(eng, ret, n_queries=16 * world * 6, lanes=16, seed=3, question_pool=24)
    wl.sessions = wl.sessions[rank::world]
    px = PeerExchange(kv)
    firsts, peer = [], []
    if pipelined:
        it = wl.rotations_with_decode(ROT, 4, peer=px) if decode else wl.rotations(ROT, peer=px)
        for r in it:
            firsts += r.first_tokens
            peer.append(kv.peer_hits())
    else:
        for _ in range(ROT):
            px.epoch_begin()
            r = wl.rotation_with_decode(4) if decode else wl.rotation()
            px.epoch_end()
            firsts += r.first_tokens
            peer.append(kv.peer_hits())
    torch.cuda.synchronize()
    dist.barrier()
    out = (kv.counters(), kv.peer_hits(), firsts, kv.free_pages())
    eng.close() if hasattr(eng, "close") else None
    del eng
    kv.close()
    return out


results = [(run(False), run(True)), (run(False, decode=True), run(True, decode=True))]
res = [None] * world
dist.all_gather_object(res, results)
if rank == 0:
    for q, (s, p) in [(q, sp) for q, rr in enumerate(res) for sp in rr]:
        assert s[0] == p[0], (q, s[0], p[0])
        if CAP <= 224:
            assert sum(s[0]["evictions_by_tier"]) > 0, s[0]
        assert s[1] > 0 and p[1] > 0, (q, s[1], p[1])
        assert len(s[2]) == len(p[2]) and len(s[2]) > 0
        agree = sum(a == b for a, b in zip(s[2], p[2])) / len(s[2])
        assert agree >= 0.97, (q, agree)
        print(f"rank {q}: counters {s[0]} peer hits seq {s[1]} pipelined {p[1]} "
              f"first-token agreement {agree:.4f} free pages {s[3]} / {p[3]}", flush=True)
    print("peer_pipeline_check ok", flush=True)
dist.destroy_process_group()
