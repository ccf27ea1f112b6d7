"""Multi-GPU plumbing for the query-sharded hot path.

One process per GPU (torch.distributed for the control plane only).  Queries are independent:
rank r serves queries i with i % N == r.  The one exchange step is the cross-GPU prefix hit: at
every epoch (= one rotation of the round-robin) each rank publishes the (block id, page) pairs of
its resident blocks; a rank's engine then serves a missed run of blocks that a peer holds by
copying the pages over NVLink (K4) instead of recomputing them.  Pages named in an epoch's
directory stay valid for the whole epoch because every rank runs its pool in epoch mode (evicted
pages are released only after the epoch-end barrier).
"""
from __future__ import annotations

import numpy as np


def shard(items, rank: int, world: int):
    """Deterministic query -> rank map: item i goes to rank i % world."""
    return items[rank::world]


def affinity_rank(key: str, world: int) -> int:
    """Prefix-affinity routing: a query goes to fnv1a(question) % world, so every
    repetition of a question — and with it the whole chain of blocks its sessions build — lands
    on the GPU that already caches it (local hits instead of NVLink peer copies)."""
    h = 14695981039346656037
    for b in key.encode():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h % world


def shard_by_affinity(items, rank: int, world: int, key=lambda x: x):
    """The items whose affinity rank is `rank`, in their original order."""
    return [x for x in items if affinity_rank(key(x), world) == rank]


def merge_directories(snapshots, rank: int):
    """snapshots[q] = (ids uint64[n_q], pages int32[n_q]) of rank q.  Returns the directory a
    given rank installs: every other rank's residents, lower rank first for duplicated ids."""
    ids, peers, pages = [], [], []
    for q, (i, p) in enumerate(snapshots):
        if q == rank or len(i) == 0:
            continue
        ids.append(np.asarray(i, dtype=np.uint64))
        pages.append(np.asarray(p, dtype=np.int32))
        peers.append(np.full(len(i), q, dtype=np.int32))
    if not ids:
        return (np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.int32))
    return np.concatenate(ids), np.concatenate(peers), np.concatenate(pages)


class PeerExchange:
    """Wires a rank's KvCacheState to its peers and runs the per-epoch directory exchange."""

    def __init__(self, kv, group=None, use_ipc=True):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.kv = kv
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world > 1 and use_ipc:
            handles = [None] * self.world
            dist.all_gather_object(handles, kv.ipc_handle(), group=group)
            for q, h in enumerate(handles):
                if q != self.rank:
                    kv.attach_peer(q, h)
        kv.set_epoch_mode(True)

    def epoch_begin(self):
        """Barrier, then exchange resident snapshots and install the merged directory."""
        snap = self.kv.resident_ids_pages()
        snaps = [None] * self.world
        self.dist.all_gather_object(snaps, snap, group=self.group)
        ids, peers, pages = merge_directories(snaps, self.rank)
        self.kv.set_peer_directory(ids, peers, pages)
        return len(ids)

    def epoch_end(self):
        """After this rank's epoch work completed on the device: wait for every rank, then the
        pages evicted during the epoch may be reused."""
        self.dist.barrier(group=self.group)
        self.kv.release_deferred()
        self._pending = None
        self._marks = []

    # ---- pipelined epochs (GraphCoTWorkload.rotations: the bookkeeping of rotation r+1 runs
    # while the forward of rotation r is on the GPU).  Residents at the moment a rotation's
    # bookkeeping starts (snapshot S_e, rotations < e) are only complete on the device once
    # forward e-1 has finished, so S_e is published after that wait and serves the bookkeeping
    # of rotation e+1 (one rotation later than the sequential protocol).  A page evicted after
    # S_e was taken may still be named by S_e: it stays deferred until every rank has finished
    # the forward that consumed S_e's directory (rotation e+1), i.e. it is released at the
    # exchange after wait(e+1).  Cache decisions do not depend on the directory (peer hits only
    # change computed -> copied), so the lag changes no counter.
    def before_bookkeeping(self):
        """Call right before a rotation's prefill bookkeeping: snapshot + deferral mark."""
        self._pending = (self.kv.resident_ids_pages(), self.kv.defer_mark())

    def after_wait(self):
        """Call after the oldest in-flight rotation's forward completed: publish the snapshot
        taken before the next rotation's bookkeeping (now complete on the device), install the
        merged directory, release the pages deferred before the previous snapshot's mark."""
        snap, mark = self._pending if getattr(self, "_pending", None) else (
            (np.zeros(0, np.uint64), np.zeros(0, np.int32)), self.kv.defer_mark())
        snaps = [None] * self.world
        self.dist.all_gather_object(snaps, snap, group=self.group)  # also a barrier
        ids, peers, pages = merge_directories(snaps, self.rank)
        self.kv.set_peer_directory(ids, peers, pages)
        marks = getattr(self, "_marks", [])
        if marks:
            self.kv.release_deferred_before(marks[-1])
        self._marks = [mark]
        return len(ids)
