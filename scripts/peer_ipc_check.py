"""torchrun --nproc-per-node 2: two ranks (both on cuda:0 here; one per GPU in production)
exchange their KV pools by CUDA IPC and run two epochs: rank 0 computes a prompt, rank 1 then
prefills the same prompt and must serve its blocks from rank 0's pool (peer copies), with logits
equal to rank 0's."""
import os
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.sharding import PeerExchange  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
dev = int(os.environ.get("GLMX_PEER_DEVICE", "0"))
cfg = glmx.TINY
model = glmx.Model(cfg, dev)
kv = glmx.KvCacheState(128, 16, glmx.PRIORITY, device=dev, n_layers=cfg.n_layers,
                       n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, headroom_pages=128)
eng = glmx.Engine(model, kv, max_requests=4, max_batch_tokens=1024, max_decode=4, max_context=1024)
ex = PeerExchange(kv)
prompt = [f"w{i}" for i in range(200)]
req = glmx.Request(prompt, [(0, 40, 0), (40, 200, 1)], f"s{rank}")

ex.epoch_begin()  # epoch 0: nobody has anything
logits0 = None
if rank == 0:
    _, _, logits0 = eng.prefill([req], want_logits=True)
ex.epoch_end()

ex.epoch_begin()  # epoch 1: rank 1 sees rank 0's 12 blocks
logits1 = None
if rank == 1:
    _, _, logits1 = eng.prefill([req], want_logits=True)
ex.epoch_end()
res = [None, None]
dist.all_gather_object(res, (kv.peer_hits(), logits0 if rank == 0 else logits1))
if rank == 0:
    hits1 = res[1][0]
    d = float(np.abs(res[0][1] - res[1][1]).max())
    assert hits1 == 12, hits1
    assert d < 2e-2, d
    print("peer_ipc_check ok", hits1, d, flush=True)
dist.destroy_process_group()
