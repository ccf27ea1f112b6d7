"""Multi-process host logic of the query-sharded path on CPU (gloo, world_size 2): query sharding,
the per-epoch resident-directory exchange, and the merged directory each rank installs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_01633_b200.sharding import merge_directories, shard


def test_shard_is_a_partition():
    items = list(range(103))
    parts = [shard(items, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == items
    assert all(i % 4 == r for r, p in enumerate(parts) for i in p)


def test_merge_directories_excludes_self_and_keeps_rank_order():
    snaps = [(np.array([1, 2], np.uint64), np.array([10, 11], np.int32)),
             (np.array([2, 3], np.uint64), np.array([20, 21], np.int32)),
             (np.array([], np.uint64), np.array([], np.int32))]
    ids, peers, pages = merge_directories(snaps, 1)
    assert ids.tolist() == [1, 2] and peers.tolist() == [0, 0] and pages.tolist() == [10, 11]
    ids, peers, pages = merge_directories(snaps, 2)
    assert ids.tolist() == [1, 2, 2, 3] and peers.tolist() == [0, 0, 1, 1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2511_01633_b200 as glmx
    from paper_2511_01633_b200.sharding import PeerExchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kv = glmx.KvCacheState(64, 16)  # bookkeeping-only pool handle (no device)
        queries = shard([f"q{i}" for i in range(10)], rank, world)
        for qid in queries:
            toks = ["shared"] * 32 + [qid] * 20
            kv.prefill(toks, [(0, 32, 0), (32, 52, 3)], qid)
        ex = PeerExchange(kv, use_ipc=False)
        n_dir = ex.epoch_begin()
        mine = kv.resident_ids_pages()[0]
        everyone = [None] * world
        dist.all_gather_object(everyone, sorted(int(x) for x in mine))
        others = sum((e for r, e in enumerate(everyone) if r != rank), [])
        ex.epoch_end()
        q.put((rank, len(queries), n_dir, len(others), kv.counters()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_directory_exchange():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    assert [r[1] for r in res] == [5, 5]            # 10 queries split 5/5
    for rank, n_q, n_dir, n_other, counters in res:
        assert n_dir == n_other                      # directory == every other rank's residents
        # 52 tokens = 2 shared blocks + 1 per-query block + a 4-token tail: each rank computes the
        # shared blocks once (independent caches, as G reference KvCacheStates would)
        assert counters["misses"] == 2 + n_q and counters["hits"] == 2 * (n_q - 1)


def test_affinity_routing_keeps_repeats_together():
    from paper_2511_01633_b200.sharding import affinity_rank, shard_by_affinity

    qs = [f"Which item is linked from all of: v{i % 37}; v{(i * 7) % 37}?" for i in range(400)]
    for world in (2, 4, 8):
        parts = [shard_by_affinity(list(range(len(qs))), r, world, key=lambda i: qs[i])
                 for r in range(world)]
        assert sorted(sum(parts, [])) == list(range(len(qs)))      # a partition
        owner = {}
        for r, p in enumerate(parts):
            for i in p:
                assert owner.setdefault(qs[i], r) == r              # repeats share a rank
        assert all(affinity_rank(q, world) == owner[q] for q in qs)
        assert min(len(p) for p in parts) > 0
