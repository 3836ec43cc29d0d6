"""Multi-GPU sharding of the feedback step: one process per GPU,
``torch.distributed`` for the plumbing.

The batch is partitioned into contiguous exec ranges in rank order; the only
exchange step is ONE allgather of the per-rank novelty deltas (S bytes per rank,
NCCL over NVLink/NVSwitch on GPUs).  Everything else is rank-local:

    scan   (rank-local)   signatures, nnz, delta D_r = class bits not in V0
    allgather(D_r)        R x S bytes
    resolve (rank-local)  exact Admit codes against P_r = V0 | OR_{q<r} D_q, then the
                          ordered merge virgin = V0 | D_0 | ... | D_{R-1}
                          (bitwise OR in the reference's polarity == AFL's AND-merge)

Exactness: the sequential virgin before global exec i is V0 | OR_{j<i} classed_j;
maps with no novelty versus V0 contribute nothing, so the state at rank r's first
exec is exactly P_r, and the rank-local first-occurrence resolve reproduces the
single-rank sequential Admit codes (checked against the oracle in
tests/test_sharding_gloo.py on CPU and tests/test_feedback_gpu.py on the GPU).

The module is backend-agnostic: ``engine`` is anything with ``feedback_scan`` /
``feedback_resolve`` (``api.Context`` in production).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous exec range [start, start+count) of `rank`; earlier ranks take the remainder."""
    per, rem = divmod(n_total, world)
    start = rank * per + min(rank, rem)
    return start, per + (1 if rank < rem else 0)


class ShardedFeedback:
    """exchange = "allgather" (default): one all_gather_into_tensor of the deltas per step (NCCL).
    exchange = "peers": every rank's delta lives in a buffer the library exports over CUDA IPC
    (hfz_peer_alloc / hfz_peer_open, handles exchanged once through the process group); the merge kernel
    of each rank loads the R deltas straight from their owners -- same device, or NVLink / NVSwitch peers --
    (hfz_feedback_resolve_peers), bracketed by two barriers of the group: no collective on the data path,
    no staging copy."""

    def __init__(self, engine, group=None, exchange: str = "allgather"):
        self.engine = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._deltas = None
        self.exchange = exchange
        self._peer_ptrs = None
        if exchange == "peers" and self.world > 1:
            S = engine.S
            self._own_ptr, handle = engine.peer_alloc(S)
            handles = [None] * self.world
            dist.all_gather_object(handles, handle, group=group)
            self._peer_ptrs = [self._own_ptr if q == self.rank else engine.peer_open(handles[q]) for q in range(self.world)]
            self._delta_buf = engine.device_view(self._own_ptr, S)
            dist.barrier(group=group)  # every rank has mapped every buffer before anyone writes or frees

    def close(self):
        """Unmap the peers' buffers and free this rank's (after a barrier: nobody still reads it)."""
        if self._peer_ptrs is not None:
            torch.cuda.synchronize()
            for q, p in enumerate(self._peer_ptrs):
                if q != self.rank:
                    self.engine.peer_close(p)
            dist.barrier(group=self.group)
            self.engine.peer_free(self._own_ptr)
            self._peer_ptrs = None

    def _meet(self):
        torch.cuda.current_stream().synchronize()  # this rank's kernels are done ...
        dist.barrier(group=self.group)             # ... and so are everybody else's

    def step(self, raw_local: torch.Tensor, virgin: torch.Tensor, edge_counts: torch.Tensor,
             out: dict | None = None):
        """One campaign iteration on this rank's shard.  `virgin`/`edge_counts` are the
        replicated campaign state (identical on all ranks before and after)."""
        if self._peer_ptrs is not None:
            out = dict(out or {})
            out["delta"] = self._delta_buf              # the scan writes this rank's delta in place
            o = self.engine.feedback_scan(raw_local, virgin, out=out)
            self._meet()                                # every rank's delta is complete
            o["admit"] = self.engine.feedback_resolve_peers(raw_local, virgin, edge_counts, self._peer_ptrs,
                                                            self.rank, admit=o.get("admit"))
            self._meet()                                # nobody overwrites a delta that is still being read
            return o
        if self.world == 1:  # nothing to exchange: the single-rank fold (scan, then one pass over the table)
            return self.engine.feedback_batch(raw_local, virgin, edge_counts, out=out)
        o = self.engine.feedback_scan(raw_local, virgin, out=out)
        delta = o["delta"]
        if self._deltas is None or self._deltas.numel() != self.world * delta.numel():
            self._deltas = torch.empty(self.world * delta.numel(), dtype=delta.dtype, device=delta.device)
        deltas = self._deltas
        dist.all_gather_into_tensor(deltas, delta, group=self.group)
        o["admit"] = self.engine.feedback_resolve(raw_local, virgin, edge_counts, deltas, self.world,
                                                  self.rank, admit=o.get("admit"))
        return o
