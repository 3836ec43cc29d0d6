"""Worker of tests/test_sharding_peers_gpu.py: one of R processes sharing GPU 0.  Every rank folds its shard of a
batch through ShardedFeedback(exchange="peers") -- deltas in CUDA IPC buffers mapped into every process, read in
place by hfz_feedback_resolve_peers -- and checks its Admit codes, the final virgin map and the edge counters
against the single-rank fold of the WHOLE batch computed on the same device."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth
from paper_2603_12485_b200.sharding import ShardedFeedback, shard_range


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    S = 65536
    ctx = hfz.Context(0, S)
    eng = ShardedFeedback(ctx, exchange="peers")
    assert eng._peer_ptrs is not None and len(eng._peer_ptrs) == world
    # per rank: the fused small step (scan / resolve halves), the pipelined and the lane-per-map kernels, and a batch
    # smaller than the world (a rank with no exec at all)
    for n_total, seed in ((world * 300 + 1, 5), (world * 5000, 6), (world * 9000 + 7, 8), (2, 7)):
        raw = torch.from_numpy(synth.maps_campaign(n_total, S, seed=seed)).to(dev)
        # single-rank truth, two steps (the second from the state the first left)
        v1, c1 = ctx.new_virgin(), ctx.new_edge_counts()
        want = [ctx.feedback_batch(raw, v1, c1)["admit"].clone() for _ in range(2)]
        start, cnt = shard_range(n_total, world, rank)
        mine = raw[start * ctx.rec:(start + cnt) * ctx.rec]
        v, c = ctx.new_virgin(), ctx.new_edge_counts()
        for it in range(2):
            o = eng.step(mine, v, c)
            assert torch.equal(o["admit"], want[it][start:start + cnt]), f"rank {rank}: Admit codes differ (n={n_total}, step {it})"
        assert torch.equal(v, v1) and torch.equal(c, c1), f"rank {rank}: virgin map / counters differ (n={n_total})"
        if n_total > 100:
            assert int((want[0] != 0).sum()) > 0
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()
    print(f"rank {rank}: ok", flush=True)


if __name__ == "__main__":
    main()
