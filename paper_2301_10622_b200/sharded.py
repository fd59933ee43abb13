"""Document sharding across GPUs: one process per GPU, one exchange step.

Shard r of W holds the documents with global id g, g % W == r, under the local id g // W.  Every shard
scores the whole query batch against its documents; the per-shard top-k' lists are all-gathered once
(NCCL over NVLink/NVSwitch: B * k' * 8 bytes per GPU — or, with a `PeerGather`, stored by each shard's
select kernel straight into every shard's buffer over peer-mapped memory, no collective launch), merged into the global V on every rank, re-ranked
by their owners, and the per-shard top-k lists gathered and merged again.  The global top-k' is contained
in the union of the shards' top-k', so the result equals the unsharded search of the same documents
(scores within the fp32 summation-order tolerance, R7).

This module holds no arithmetic: scoring, merging and re-ranking are the library's kernels
(sinn_search_stage1, sinn_merge_topk, sinn_rerank); the collective is torch.distributed's.  The protocol
is split into phases so that a test can drive W shards of one process in lockstep (`search_lockstep`)
without ranks that wait on each other.
"""
from __future__ import annotations

import numpy as np


def owner(gids, world: int):
    """Shard of each global id (numpy)."""
    return np.asarray(gids, dtype=np.int64) % world


def route_rows_host(indptr, indices, values, ids, world: int, rank: int):
    """Host-side routing of an insert batch (CSR + global ids) to shard `rank`: the rows with
    id % world == rank, re-based, with their local ids id // world.  Data movement only."""
    indptr = np.asarray(indptr, dtype=np.int64)
    ids = np.asarray(ids).astype(np.int64)
    rows = np.nonzero(ids % world == rank)[0]
    lens = indptr[rows + 1] - indptr[rows]
    out_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(lens, out=out_ptr[1:])
    # entry e of output row r comes from indptr[rows[r]] + (e - out_ptr[r])
    take = np.repeat(indptr[rows] - out_ptr[:-1], lens) + np.arange(out_ptr[-1], dtype=np.int64)
    return (out_ptr, np.asarray(indices, dtype=np.int32)[take], np.asarray(values, dtype=np.float32)[take],
            (ids[rows] // world).astype(np.uint32))


class _TorchOps:
    """The device ends of the exchange: the library's kernels."""

    @staticmethod
    def merge_topk(ids, scores, kout, id_mul=1, id_add=None):
        from . import merge_topk
        return merge_topk(ids, scores, kout, id_mul, id_add)


class PeerGather:
    """Gather buffers every shard's select kernel stores into directly (sinn_search_stage1_gather): shard r
    owns ids[r] / scores[r], [W, nq, k'] each; the other entries are peer-mapped views of the other GPUs'
    buffers (torch symmetric memory: NVLink P2P mappings), or plain local tensors when all the shards
    live in one process (tests).  Two buffer sets alternate by batch, so a shard that is one batch ahead
    never overwrites rows a slower shard is still merging; `barrier` orders the stores before the reads."""

    def __init__(self, ids_sets, scores_sets, barrier):
        self.ids_sets, self.scores_sets, self.barrier = ids_sets, scores_sets, barrier
        self.turn = 0

    def next_set(self):
        i = self.turn
        self.turn ^= 1
        return self.ids_sets[i], self.scores_sets[i]

    @classmethod
    def symmetric(cls, rank: int, world: int, nq: int, kprime: int, device, group=None):
        """Symmetric-memory buffers over the process group (one process per GPU; needs P2P access)."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        group = group or dist.group.WORLD
        shape = (2, world, nq, kprime)
        ti = symm.empty(shape, dtype=torch.int32, device=device)
        ts = symm.empty(shape, dtype=torch.float32, device=device)
        hi, hs = symm.rendezvous(ti, group), symm.rendezvous(ts, group)
        pi = [hi.get_buffer(r, shape, torch.int32) for r in range(world)]
        ps = [hs.get_buffer(r, shape, torch.float32) for r in range(world)]
        return cls([[b[i] for b in pi] for i in (0, 1)], [[b[i] for b in ps] for i in (0, 1)],
                   lambda: hi.barrier(channel=0))

    @classmethod
    def local(cls, world: int, nq: int, kprime: int, device):
        """One process, W shards on one device: the "peers" are local tensors; returns one PeerGather per
        shard sharing the same buffers (no barrier: the caller runs the shards in lockstep)."""
        import torch
        bi = [[torch.full((world, nq, kprime), -2, dtype=torch.int32, device=device) for _ in range(world)]
              for _ in (0, 1)]
        bs = [[torch.full((world, nq, kprime), float("nan"), dtype=torch.float32, device=device)
               for _ in range(world)] for _ in (0, 1)]
        return [cls(bi, bs, lambda: None) for _ in range(world)]


class ShardedIndex:
    """One shard (this rank's documents) of a document-sharded Sinnamon index.

    `index` is this rank's `paper_2301_10622_b200.Index` (or any object with its `search_stage1`,
    `rerank`, `insert_host`, `delete_host` methods); `group` a torch.distributed process group (None: the
    default group, or a single shard when torch.distributed is not initialised)."""

    def __init__(self, index, rank: int | None = None, world: int | None = None, group=None, ops=None,
                 peer: PeerGather | None = None):
        self.index = index
        self.group = group
        self.peer = peer  # stage-1 rows stored into every shard's buffer by the select kernel (no all-gather)
        if rank is None or world is None:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                rank, world = dist.get_rank(group), dist.get_world_size(group)
            else:
                rank, world = 0, 1
        self.rank, self.world = int(rank), int(world)
        self.ops = ops or _TorchOps()

    # ------------------------------------------------------------ routing (data movement only)
    def insert_host(self, indptr, indices, values, ids) -> int:
        """Insert this rank's rows of a global batch (every rank passes the same batch).  Returns the
        number of rows this shard took."""
        p, ix, v, lid = route_rows_host(indptr, indices, values, ids, self.world, self.rank)
        if lid.size:
            self.index.insert_host(p, ix, v, lid)
        return int(lid.size)

    def delete_host(self, ids) -> int:
        ids = np.asarray(ids).astype(np.int64)
        mine = ids[ids % self.world == self.rank] // self.world
        if mine.size:
            self.index.delete_host(mine.astype(np.uint32))
        return int(mine.size)

    # ------------------------------------------------------------ the search protocol, by phase
    def phase_stage1(self, q, kprime: int):
        """Local S0-S2: this shard's top-k' (LOCAL ids, approximate scores), [nq, k']."""
        return self.index.search_stage1(*q, kprime)

    def phase_stage1_gather(self, q, kprime: int):
        """Local S0-S2 whose select kernel stores this shard's rows into slot `rank` of EVERY shard's gather
        buffer (peer stores).  Returns this shard's own buffers [W, nq, k'], complete once every shard has
        passed the barrier."""
        ids, scores = self.peer.next_set()
        self.index.search_stage1_gather(*q, kprime, self.rank, ids, scores)
        return ids[self.rank], scores[self.rank]

    def phase_select(self, gathered_ids, gathered_scores, kout: int):
        """Global V from the gathered [W, nq, k'] lists (local ids -> global), identical on every rank."""
        return self.ops.merge_topk(gathered_ids, gathered_scores, kout, self.world, np.arange(self.world))

    def phase_rerank(self, q, v_ids, k: int):
        """Owner re-rank: exact scores of the candidates of V this shard holds; its top-k (global ids)."""
        return self.index.rerank(*q, v_ids, k, self.world, self.rank)

    def phase_final(self, gathered_ids, gathered_scores, k: int):
        """Top-k of the gathered per-shard top-k lists (ids are global already)."""
        return self.ops.merge_topk(gathered_ids, gathered_scores, k, 1, None)

    def all_gather(self, t):
        """[...] -> [W, ...] over the group (a view for a single shard)."""
        if self.world == 1:
            return t.unsqueeze(0)
        import torch
        import torch.distributed as dist
        # (the output is the concatenation along dim 0, rank-major: the [W, ...] view of it)
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out.view((self.world,) + tuple(t.shape))

    def search(self, q_indptr, q_indices, q_values, k: int, kprime: int, rerank: bool = True):
        """Sharded sinn_search: every rank passes the same query batch and receives the same
        (global ids int32 [nq, k], scores float32 [nq, k])."""
        q = (q_indptr, q_indices, q_values)
        if self.peer is not None and self.world > 1:
            gi, gs = self.phase_stage1_gather(q, kprime)
            self.peer.barrier()
        else:
            ci, cs = self.phase_stage1(q, kprime)
            gi, gs = self.all_gather(ci), self.all_gather(cs)
        if not rerank:
            return self.phase_select(gi, gs, k)
        vi, _ = self.phase_select(gi, gs, kprime)
        li, ls = self.phase_rerank(q, vi, k)
        return self.phase_final(self.all_gather(li), self.all_gather(ls), k)


def search_lockstep(shards, q, k: int, kprime: int, rerank: bool = True, stack=None):
    """Drive the W shards of ONE process through the protocol phase by phase, with a stack of the
    per-shard outputs in place of the all-gather (tests: W indexes on one GPU, no rank ever waits on
    another).  Returns every shard's result (they must agree)."""
    if stack is None:
        import torch
        stack = torch.stack
    if shards[0].peer is not None:  # every shard stores its rows into all the buffers; no stack
        own = [s.phase_stage1_gather(q, kprime) for s in shards]
        if not rerank:
            return [s.phase_select(own[r][0], own[r][1], k) for r, s in enumerate(shards)]
        V = [s.phase_select(own[r][0], own[r][1], kprime) for r, s in enumerate(shards)]
    else:
        s1 = [s.phase_stage1(q, kprime) for s in shards]
        gi, gs = stack([a for a, _ in s1]), stack([b for _, b in s1])
        if not rerank:
            return [s.phase_select(gi, gs, k) for s in shards]
        V = [s.phase_select(gi, gs, kprime) for s in shards]
    loc = [s.phase_rerank(q, V[r][0], k) for r, s in enumerate(shards)]
    ai, as_ = stack([a for a, _ in loc]), stack([b for _, b in loc])
    return [s.phase_final(ai, as_, k) for s in shards]
