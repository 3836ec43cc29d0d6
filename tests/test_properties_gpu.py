"""Size-independent properties at BASELINE.json's full sizes (the oracle only checks samples here):
idempotence and order-independence of the virgin fold, sharded == single-rank at 65,536 execs,
signatures against the oracle on a sample, counter conservation of the edge-record stage."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

pytestmark = pytest.mark.gpu
S = 65536
REC = synth.record_bytes(S)
N_FULL = 65536  # configs[1]


@pytest.fixture(scope="module")
def full_batch():
    """configs[1]: 65,536 campaign-like maps on the device (10.7 GB) + the virgin warmed with 4,096."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = torch.device("cuda", 0)
    raw = torch.empty(N_FULL * REC, dtype=torch.uint8, device=dev)
    for i in range(0, N_FULL, 4096):
        raw[i * REC:(i + 4096) * REC] = torch.from_numpy(synth.maps_campaign(4096, S, first=i, p_extra=64, p_rare=64)).to(dev)
    ctx = hfz.Context(0, S)
    v0, c0 = ctx.new_virgin(), ctx.new_edge_counts()
    ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(4096, S, first=1 << 24)).to(dev), v0, c0)
    ctx.synchronize()
    yield ctx, raw, v0, c0
    ctx.close()
    del raw


def fold(ctx, raw, v0, c0):
    v, c = v0.clone(), c0.clone()
    o = ctx.feedback_batch(raw, v, c)
    ctx.synchronize()
    return {k: t.clone() for k, t in o.items()}, v, c


def test_fold_is_idempotent_at_full_size(full_batch):
    ctx, raw, v0, c0 = full_batch
    o1, v1, c1 = fold(ctx, raw, v0, c0)
    assert int((o1["admit"] != 0).sum()) > 100           # the batch does discover things
    o2, v2, c2 = fold(ctx, raw, v1, c1)
    assert int((o2["admit"] != 0).sum()) == 0            # nothing is new the second time
    assert torch.equal(v1, v2) and torch.equal(c1, c2)
    assert torch.equal(o1["sig_full"], o2["sig_full"]) and torch.equal(o1["sig_simple"], o2["sig_simple"])
    assert torch.equal(o1["nnz"], o2["nnz"])
    # virgin only grows, and the counters count exactly the slots that turned non-zero
    assert bool(((v1 & v0) == v0).all())
    H = S // 2
    grown = (v1 != 0) & (v0 == 0)
    assert int(grown[:H].sum()) == int(c1[0] - c0[0]) and int(grown[H:].sum()) == int(c1[1] - c0[1])


def test_final_virgin_is_order_independent_at_full_size(full_batch):
    ctx, raw, v0, c0 = full_batch
    o1, v1, c1 = fold(ctx, raw, v0, c0)
    g = torch.Generator(device="cpu")
    g.manual_seed(5)
    perm = torch.randperm(N_FULL, generator=g).to(raw.device)
    shuffled = raw.view(N_FULL, REC)[perm].contiguous().view(-1)
    o2, v2, c2 = fold(ctx, shuffled, v0, c0)
    assert torch.equal(v1, v2) and torch.equal(c1, c2)
    assert torch.equal(o1["sig_full"][perm], o2["sig_full"])     # a signature belongs to its map alone
    assert torch.equal(o1["sig_simple"][perm], o2["sig_simple"])
    # checksum of checksums
    x1 = np.bitwise_xor.reduce(o1["sig_full"].cpu().numpy().view(np.uint64))
    x2 = np.bitwise_xor.reduce(o2["sig_full"].cpu().numpy().view(np.uint64))
    assert x1 == x2
    del shuffled


def test_sharded_fold_equals_single_rank_at_full_size(full_batch):
    """configs[4] shape on one GPU: 4 simulated ranks x 16,384 execs, allgather of the deltas,
    rank-ordered resolve -- Admit codes, signatures, virgin and counters equal the single fold."""
    ctx, raw, v0, c0 = full_batch
    o1, v1, c1 = fold(ctx, raw, v0, c0)
    R, per = 4, N_FULL // 4
    ctxs = [hfz.Context(0, S) for _ in range(R)]
    try:
        shards = [raw[r * per * REC:(r + 1) * per * REC] for r in range(R)]
        scans = [ctxs[r].feedback_scan(shards[r], v0) for r in range(R)]
        deltas = torch.cat([s["delta"] for s in scans])
        admits = []
        for r in range(R):
            v, c = v0.clone(), c0.clone()
            admits.append(ctxs[r].feedback_resolve(shards[r], v, c, deltas, R, r))
            ctxs[r].synchronize()
            assert torch.equal(v, v1) and torch.equal(c, c1), f"rank {r} state differs"
        assert torch.equal(torch.cat(admits), o1["admit"])
        assert torch.equal(torch.cat([s["sig_full"] for s in scans]), o1["sig_full"])
        # the peer-memory form: each rank's merge reads the four deltas where the scans left them
        peer_deltas = [s["delta"] for s in scans]
        admits2 = []
        for r in range(R):
            v, c = v0.clone(), c0.clone()
            admits2.append(ctxs[r].feedback_resolve_peers(shards[r], v, c, peer_deltas, r))
            ctxs[r].synchronize()
            assert torch.equal(v, v1) and torch.equal(c, c1), f"rank {r} state differs (peers)"
        assert torch.equal(torch.cat(admits2), o1["admit"])
    finally:
        for c in ctxs:
            c.close()


def test_signatures_and_admits_against_the_oracle_on_a_sample(full_batch, checker):
    ctx, raw, v0, c0 = full_batch
    o1, _, _ = fold(ctx, raw, v0, c0)
    # signatures of a scattered sample; Admit codes of the first 2,048 execs (sequential prefix)
    idx = torch.arange(0, N_FULL, 257, device=raw.device)
    sample = raw.view(N_FULL, REC)[idx].contiguous().cpu().numpy().reshape(-1)
    vv, cc = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    want = checker.feedback_batch(sample, idx.numel(), S, vv, cc)
    assert np.array_equal(o1["sig_full"][idx].cpu().numpy().view(np.uint64), want["sig_full"])
    assert np.array_equal(o1["sig_simple"][idx].cpu().numpy().view(np.uint64), want["sig_simple"])
    assert np.array_equal(o1["nnz"][idx].cpu().numpy().view(np.uint32), want["nnz"])
    pre = raw[: 2048 * REC].cpu().numpy()
    vv, cc = v0.cpu().numpy().copy(), c0.cpu().numpy().view(np.uint64).copy()
    want = checker.feedback_batch(pre, 2048, S, vv, cc)
    assert np.array_equal(o1["admit"][:2048].cpu().numpy(), want["admit"])


def test_edge_record_conserves_bumps(ctx):
    """configs[2] trace shape: every bump adds one to exactly one counter (no counter saturates
    here), so an exec's counters sum to its warp_edge_events; and the stage is deterministic."""
    n = 96
    tr = synth.bb_traces(n, seed=44)
    i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(ctx.device)
    args = (i64(tr["launch_off"]), torch.from_numpy(np.ascontiguousarray(tr["dims"], np.uint32).view(np.int32)).to(ctx.device),
            i64(tr["thread_off"]), i64(tr["ev_off"]),
            torch.from_numpy(np.ascontiguousarray(tr["sites"], np.uint32).view(np.int32)).to(ctx.device))
    raw1, ev1 = ctx.edge_record_batch(*args, n)
    raw2, ev2 = ctx.edge_record_batch(*args, n)
    ctx.synchronize()
    assert torch.equal(raw1, raw2) and torch.equal(ev1, ev2)
    dev_half = raw1.view(n, REC)[:, S // 2:].contiguous().view(torch.int32).to(torch.int64)
    assert torch.equal(dev_half.sum(dim=1), ev1)
    assert int(ev1.min()) > 0


def test_one_large_fold_equals_two_half_folds(full_batch):
    """A batch larger than configs[1] (2 x 65,536 execs = 21 GB: every warp of the throughput kernel
    walks several groups) folded in ONE call equals folding its halves one after the other."""
    ctx, raw, v0, c0 = full_batch
    dev = raw.device
    second = torch.empty_like(raw)
    for i in range(0, N_FULL, 4096):
        second[i * REC:(i + 4096) * REC] = torch.from_numpy(
            synth.maps_campaign(4096, S, first=N_FULL + i, p_extra=64, p_rare=64)).to(dev)
    both = torch.cat([raw, second])
    o_all, v_all, c_all = fold(ctx, both, v0, c0)
    o1, v1, c1 = fold(ctx, raw, v0, c0)
    o2, v2, c2 = fold(ctx, second, v1, c1)
    assert torch.equal(v_all, v2) and torch.equal(c_all, c2)
    for k in ("admit", "sig_full", "sig_simple", "nnz"):
        assert torch.equal(o_all[k], torch.cat([o1[k], o2[k]])), k
    assert int((o2["admit"] != 0).sum()) > 0
    del both, second
