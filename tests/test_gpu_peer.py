"""Cross-GPU prefix hits on one B200: a second engine with its own pool serves the
missed blocks another pool holds by K4 page copies instead of recomputing them.  Bookkeeping
stays the reference's (those blocks are misses); the logits equal the fully computed ones and
the fp32 oracle.  The multi-process variant exchanges pools by CUDA IPC under torchrun (gloo for
the directory) with both ranks on cuda:0."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2511_01633_b200 as glmx
from oracle.decoder import Decoder, token_ids

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def words(n, t="w"):
    return [f"{t}{i}" for i in range(n)]


def make_pool(cfg, cap=128):
    return glmx.KvCacheState(cap, 16, glmx.PRIORITY, device=0, n_layers=cfg.n_layers,
                             n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, headroom_pages=128)


def test_peer_copy_replaces_recompute(ref):
    cfg = glmx.TINY
    model = glmx.Model(cfg, 0)
    kv_a, kv_b = make_pool(cfg), make_pool(cfg)
    ea = glmx.Engine(model, kv_a, max_requests=4, max_batch_tokens=1024, max_decode=4, max_context=1024)
    eb = glmx.Engine(model, kv_b, max_requests=4, max_batch_tokens=1024, max_decode=4, max_context=1024)
    p = words(150)
    ra, fa, la = ea.prefill([glmx.Request(p, [(0, 40, 0), (40, 150, 2)], "s")], want_logits=True)
    kv_b.attach_peer_local(0, kv_a)
    kv_b.set_epoch_mode(True)
    ids, pages = kv_a.resident_ids_pages()
    kv_b.set_peer_directory(ids, np.zeros(len(ids), np.int32), pages)
    # b first hits 0 local blocks, then the 9 blocks of a's chain are served by peer copies
    q = p[:144] + words(10, "x")
    rb, fb, lb = eb.prefill([glmx.Request(q, [(0, 40, 0), (40, 154, 1)], "t")], want_logits=True)
    assert kv_b.peer_hits() == 9
    # bookkeeping identical to an independent reference KvCacheState
    rk = oracle.RefKv(ref, 128, 16, 0)
    st, rep, ev = rk.prefill(q, [(0, 40, 0), (40, 154, 1)], "t")
    assert (rb[0].cached_tokens, rb[0].computed_tokens, rb[0].tail_tokens) == rep
    dec = Decoder(cfg, model.export_all())
    ref_l, _ = dec.forward(token_ids(q, cfg.vocab))
    err = np.abs(lb[0] - ref_l)
    assert np.all(err <= 2e-2 + 1e-2 * np.abs(ref_l)), err.max()
    kv_b.release_deferred()


def test_ipc_two_processes_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517",
           os.path.join(ROOT, "scripts", "peer_ipc_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "peer_ipc_check ok" in out.stdout


def test_pipelined_epochs_match_sequential():
    # rotation r+1's bookkeeping overlaps forward r: the directory is published one rotation
    # later and evicted pages stay deferred until every rank finished the forward that used it
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29519",
           os.path.join(ROOT, "scripts", "peer_pipeline_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "peer_pipeline_check ok" in out.stdout
