"""N > 1 path on CPU: world_size-2 gloo processes drive the host-side sharding logic
(paper_2603_12485_b200/sharding.py: contiguous partition, ONE allgather of the per-rank novelty
deltas, rank-ordered resolve) with an oracle-backed stand-in for the device engine, and the
result must equal the single-rank sequential oracle over the concatenated batch
(Admit codes per exec, final virgin, edge counters, signatures)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle
from paper_2603_12485_b200 import synth
from paper_2603_12485_b200.sharding import ShardedFeedback, shard_range

S = 65536
REC = synth.record_bytes(S)


class OracleEngine:
    """Test-only engine with the Context.feedback_scan / feedback_resolve contract, on CPU."""

    def __init__(self):
        self.port = pyoracle.Port()

    def feedback_scan(self, raw, virgin_v0, out=None):
        raw_np = raw.numpy()
        n = raw_np.size // REC
        v0 = virgin_v0.numpy()
        delta = self.port.rank_delta(raw_np, n, S, v0)
        # signatures / nnz do not depend on the virgin map
        o = self.port.feedback_batch(raw_np, n, S, v0.copy(), np.zeros(2, np.uint64))
        return dict(delta=torch.from_numpy(delta), sig_full=torch.from_numpy(o["sig_full"].view(np.int64)),
                    sig_simple=torch.from_numpy(o["sig_simple"].view(np.int64)), nnz=torch.from_numpy(o["nnz"].view(np.int32)))

    def feedback_resolve(self, raw, virgin, edge_counts, deltas, n_ranks, rank, admit=None):
        raw_np = raw.numpy()
        n = raw_np.size // REC
        d = deltas.numpy().reshape(n_ranks, S)
        v0 = virgin.numpy()
        prior = v0.copy()
        for q in range(rank):
            prior |= d[q]
        o = self.port.feedback_batch(raw_np, n, S, prior.copy(), np.zeros(2, np.uint64))
        final = v0.copy()
        for q in range(n_ranks):           # fixed rank order (OR here == AFL's AND-merge)
            final |= d[q]
        ec = edge_counts.numpy().view(np.uint64)
        turned = (v0 == 0) & (final != 0)
        ec[0] += np.count_nonzero(turned[: S // 2])
        ec[1] += np.count_nonzero(turned[S // 2:])
        virgin.copy_(torch.from_numpy(final))
        return torch.from_numpy(o["admit"])


def _worker(rank, world, port_no, raw, v0, c0, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_total = raw.size // REC
        start, cnt = shard_range(n_total, world, rank)
        local = torch.from_numpy(raw[start * REC:(start + cnt) * REC].copy())
        virgin = torch.from_numpy(v0.copy())
        counts = torch.from_numpy(c0.copy().view(np.int64))
        eng = ShardedFeedback(OracleEngine())
        # two iterations with the campaign state carried across
        half = cnt // 2
        outs = []
        for it in range(2):
            part = local[it * half * REC:(it + 1) * half * REC] if it == 0 else local[half * REC:]
            o = eng.step(part, virgin, counts)
            outs.append(o)
        q.put((rank, [o["admit"].numpy().copy() for o in outs], [o["sig_full"].numpy().view(np.uint64).copy() for o in outs],
               virgin.numpy().copy(), counts.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partition():
    for n in (0, 1, 7, 64, 65536, 524288):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == n
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


@pytest.mark.timeout(300)
def test_two_rank_gloo_equals_sequential_oracle():
    world = 2
    per = 48
    port = pyoracle.Port()
    warm = synth.maps_campaign(64, S, seed=21)
    raw = synth.maps_campaign(world * per, S, seed=21, first=64, p_extra=6, p_rare=6)
    v0, c0 = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    port.feedback_batch(warm, 64, S, v0, c0)

    # sequential ground truth in the order the sharded run folds: iteration 0 = first halves of
    # every rank's shard (rank order), iteration 1 = second halves
    half = per // 2
    order = []
    for it in range(2):
        for r in range(world):
            s = r * per + it * half
            order += list(range(s, s + half))
    seq = np.concatenate([raw[i * REC:(i + 1) * REC] for i in order])
    vv, cc = v0.copy(), c0.copy()
    want = port.feedback_batch(seq, len(order), S, vv, cc)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, pn, raw, v0, c0, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got_admit, got_sig = [], []
    for it in range(2):
        for r in range(world):
            got_admit.append(res[r][1][it])
            got_sig.append(res[r][2][it])
    assert np.array_equal(np.concatenate(got_admit), want["admit"])
    assert np.array_equal(np.concatenate(got_sig), want["sig_full"])
    for r in range(world):
        assert np.array_equal(res[r][3], vv), "virgin differs from the sequential fold"
        assert np.array_equal(res[r][4], cc), "edge counters differ"
    assert set(want["admit"].tolist()) >= {0, 2}
