"""K1 parity: batched edge record on the GPU vs the CPU oracle (and the reference runtime for
the cases it pins), counter for counter."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

pytestmark = pytest.mark.gpu
S, H = 65536, 32768


@pytest.fixture(autouse=True, params=["flat", "per_exec"])
def edge_path(request, ctx):
    """Every case runs through both K1 paths: the flat decide + count kernels (default; execs whose
    launches differ in geometry still go to the per-exec kernel) and the per-exec kernel alone."""
    ctx.set_option("edge_flat", 1 if request.param == "flat" else 0)
    yield request.param
    ctx.set_option("edge_flat", 1)


def to_dev(ctx, tr):
    i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(ctx.device)
    sites = np.ascontiguousarray(tr["sites"], np.uint32)
    if sites.size == 0:
        sites = np.zeros(1, np.uint32)
    return (i64(tr["launch_off"]), torch.from_numpy(np.ascontiguousarray(tr["dims"], np.uint32).view(np.int32)).to(ctx.device),
            i64(tr["thread_off"]), i64(tr["ev_off"]), torch.from_numpy(sites.view(np.int32)).to(ctx.device))


def run_gpu(ctx, tr, n_exec):
    lo, dims, to, eo, sites = to_dev(ctx, tr)
    raw, ev = ctx.edge_record_batch(lo, dims, to, eo, sites, n_exec)
    ctx.synchronize()
    return raw.cpu().numpy(), ev.cpu().numpy().view(np.uint64)


def pack(execs):
    """execs: list of (dims (L,6), ev_off (T+1), sites) per exec -> batch layout."""
    launch_off, dims, thread_off, ev_off, sites = [0], [], [0], [0], []
    for d, e, s in execs:
        d = np.asarray(d, np.uint32).reshape(-1, 6)
        base_ev = len(sites)
        t = 0
        for l in range(d.shape[0]):
            threads = int(np.prod(d[l].astype(np.uint64)))
            dims.append(d[l])
            thread_off.append(thread_off[-1] + threads)
        ev_off.extend((np.asarray(e, np.uint64)[1:] + base_ev).tolist())
        sites.extend(np.asarray(s, np.uint32).tolist())
        launch_off.append(launch_off[-1] + d.shape[0])
    return dict(launch_off=np.array(launch_off, np.uint64), dims=np.array(dims, np.uint32).reshape(-1, 6),
                thread_off=np.array(thread_off, np.uint64), ev_off=np.array(ev_off, np.uint64),
                sites=np.array(sites, np.uint32))


def check(ctx, port, tr, n_exec, S_=S):
    raw, ev = run_gpu(ctx, tr, n_exec)
    want_raw, want_ev = port.edge_record_batch(tr["launch_off"], tr["dims"], tr["thread_off"], tr["ev_off"],
                                               tr["sites"], n_exec, S_)
    assert np.array_equal(ev, want_ev), (ev[:8], want_ev[:8])
    assert np.array_equal(raw, want_raw)
    return raw


def chain(block, launches, grid=(1, 1, 1)):
    threads = int(np.prod(block)) * int(np.prod(grid))
    dims, ev, sites = [], [0], []
    for ch in launches:
        dims.append([*grid, *block])
        for _ in range(threads):
            sites.extend(ch)
            ev.append(len(sites))
    return (np.array(dims, np.uint32), np.array(ev, np.uint64), np.array(sites, np.uint32))


def test_reference_chains(ctx, port):
    """tests/test_hdvm.cpp:89-127 + acceptance criterion 5 as one batch."""
    execs = [chain((t, 1, 1), [[11, 29, 11, 500]]) for t in (1, 31, 32, 33, 64, 100, 1024)]
    execs.append(chain((33, 1, 1), [[7]]))
    execs.append(chain((40, 1, 1), [[3, 9]], grid=(2, 2, 1)))
    execs.append(chain((8, 1, 1), [[5, 6], [6, 5, 6]]))
    execs += [chain((t, 1, 1), [[7777]]) for t in (1, 31, 32, 33, 64, 100, 1024)]
    raw = check(ctx, port, pack(execs), len(execs))
    rec = synth.record_bytes(S)
    dev = raw.reshape(len(execs), rec)[:, H:].view(np.uint32)
    assert dev[7][7] == 2
    for k, t in enumerate((1, 31, 32, 33, 64, 100, 1024)):
        assert dev[10 + k][7777] == (t + 31) // 32


def test_divergence_and_loops(ctx, port):
    """tests/test_hdvm.cpp:129-187."""
    dims = np.array([[1, 1, 1, 32, 1, 1]], np.uint32)
    s1, e1 = [], [0]
    for t in range(32):
        s1 += [10, 999] if t == 5 else [10]
        e1.append(len(s1))
    s2, e2 = [], [0]
    for t in range(32):
        s2 += [77] * ((t % 31) + 1)
        e2.append(len(s2))
    raw = check(ctx, port, pack([(dims, e1, s1), (dims, e2, s2)]), 2)
    dev = raw.reshape(2, synth.record_bytes(S))[:, H:].view(np.uint32)
    assert dev[0][10] == 1 and dev[0][((10 >> 1) ^ 999) % 32768] == 1
    assert dev[1][77] == 1 and dev[1][(77 >> 1) ^ 77] == 30


def test_random_3d_multi_launch(ctx, port):
    from tests.test_oracle_vs_ref import random_exec
    rng = np.random.default_rng(11)
    execs = [random_exec(rng, int(rng.integers(1, 4)), three_d=bool(i % 2)) for i in range(80)]
    check(ctx, port, pack(execs), len(execs))


def test_uniform_launches_with_idle_threads(ctx, port):
    """Same geometry in every launch (one work queue across launches, prev read from the trace):
    threads that run no events in some launches must carry prev from the last launch where they
    did; 3-D geometry so the thread index <-> gtid mapping matters; divergent and coherent warps."""
    rng = np.random.default_rng(14)
    execs = []
    for ex in range(12):
        d = [2, 2, 1, 8, 3, 2] if ex % 2 else [3, 1, 1, 48, 1, 1]
        threads = int(np.prod(d))
        n_launch = int(rng.integers(2, 6))
        ev, sites = [0], []
        common = rng.integers(1, 300, 6).tolist()
        for l in range(n_launch):
            for t in range(threads):
                r = rng.random()
                if r < 0.35:
                    pass                                    # idle in this launch
                elif r < 0.75:
                    sites.extend(common[: 1 + (l % 5)])     # coherent-looking sequence
                else:
                    sites.extend(rng.integers(1, 300, int(rng.integers(1, 9))).tolist())
                ev.append(len(sites))
        execs.append((np.array([d] * n_launch, np.uint32), ev, sites))
    check(ctx, port, pack(execs), len(execs))


def test_divergent_warps_small_tables(ctx, port):
    """Divergent warps that fit the transposed replay's table (a few hundred distinct sites, at
    most 15 visits per lane and site), including the site id 0xffffffff (the table's free-row
    marker) and lanes that differ only in their last event."""
    rng = np.random.default_rng(15)
    execs = []
    for ex in range(6):
        dims = np.array([[2, 1, 1, 64, 1, 1]] * 2, np.uint32)
        pool = np.concatenate([rng.integers(0, 2 ** 32, 300, dtype=np.uint64), [0xFFFFFFFF, 0, 1]])
        ev, sites = [0], []
        for l in range(2):
            for t in range(128):
                n = int(rng.integers(0, 24))
                seq = pool[rng.integers(0, len(pool) if ex % 2 else 40, n)].tolist()
                if t % 7 == 0:
                    seq += [0xFFFFFFFF] * int(rng.integers(1, 6))
                if ex == 5:
                    seq = [5, 6, 7, 8, 9, 10 + (t % 3)]     # nearly coherent: same prefix, 3 endings
                sites.extend(int(x) for x in seq)
                ev.append(len(sites))
        execs.append((dims, ev, sites))
    check(ctx, port, pack(execs), len(execs))


def test_counts_beyond_16_bits_replay_with_wide_counters(ctx, port):
    """The shared-memory counters are 16-bit pairs; an exec whose counter comes near 65,536 is
    replayed with u32 counters in its output record.  One thread looping 70,000 times on a site,
    a warp of 32 coherent threads looping 66,000 times, next to ordinary execs."""
    dims = np.array([[1, 1, 1, 1, 1, 1]], np.uint32)
    loop1 = ([dims, [0, 70000], [4242] * 70000])
    d32 = np.array([[1, 1, 1, 32, 1, 1]], np.uint32)
    sites, ev = [], [0]
    for t in range(32):
        sites += [77, 78] * 33000
        ev.append(len(sites))
    loop32 = (d32, ev, sites)
    execs = [chain((64, 1, 1), [[1, 2, 3]]), loop1, chain((33, 1, 1), [[9, 9, 9, 10]]), loop32, chain((8, 1, 1), [[5, 6], [6, 5, 6]])]
    raw = check(ctx, port, pack(execs), len(execs))
    dev = raw.reshape(len(execs), synth.record_bytes(S))[:, H:].view(np.uint32)
    assert dev[1][4242] == 1 and dev[1][(4242 >> 1) ^ 4242] == 69999
    assert int(dev[3].max()) >= 32999


def test_many_distinct_sites_forces_partitioning(ctx, port):
    """Fully divergent warps with far more distinct sites than the per-warp table holds."""
    rng = np.random.default_rng(12)
    execs = []
    for _ in range(3):
        dims = np.array([[2, 1, 1, 64, 1, 1]], np.uint32)
        ev, sites = [0], []
        for t in range(128):
            n = int(rng.integers(20, 60))
            sites.extend(rng.integers(0, 2 ** 32, n, dtype=np.uint64).tolist())
            # plus revisits of earlier sites so the k-th visit rule matters
            sites.extend(int(sites[int(i)]) for i in rng.integers(max(0, len(sites) - 50), len(sites), 10))
            ev.append(len(sites))
        execs.append((dims, ev, sites))
    check(ctx, port, pack(execs), 3)


def test_empty_and_invalid_launches(ctx, port):
    """Threads without events, an exec without launches; reference rejects oversized launches."""
    d = np.array([[1, 1, 1, 40, 1, 1]], np.uint32)
    ev = np.zeros(41, np.uint64)
    execs = [(d, ev, []), (np.zeros((0, 6), np.uint32), [0], []), chain((16, 1, 1), [[1, 2, 3]])]
    check(ctx, port, pack(execs), 3)


def test_synthetic_config3_shape(ctx, port):
    """BASELINE.json configs[2] trace recipe (4 launches x 16x256 threads) on a few execs, then the
    fused feedback kernel on the produced maps."""
    tr = synth.bb_traces(6, seed=44)
    raw = check(ctx, port, tr, 6)
    virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
    o = ctx.feedback_batch(torch.from_numpy(raw).to(ctx.device), virgin, counts)
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    want = port.feedback_batch(raw, 6, S, v, c)
    assert np.array_equal(o["admit"].cpu().numpy(), want["admit"])
    assert np.array_equal(o["sig_full"].cpu().numpy().view(np.uint64), want["sig_full"])


def test_flat_path_in_chunks(ctx, port, edge_path):
    """A 1 MB bump-list scratch (262,144 events) cuts the batch into chunks of one exec each."""
    if edge_path != "flat":
        pytest.skip("flat path only")
    tr = synth.bb_traces(5, seed=21)
    ctx.set_option("edge_scratch_mb", 1)
    try:
        check(ctx, port, tr, 5)
    finally:
        ctx.set_option("edge_scratch_mb", 2048)


def test_flat_path_mixed_batch(ctx, port):
    """Execs the flat path takes (one launch, or equal geometries) interleaved with execs it leaves to
    the per-exec kernel (launches of differing geometry), plus launches of differing sizes so the
    flat queue is searched rather than divided."""
    from tests.test_oracle_vs_ref import random_exec
    rng = np.random.default_rng(23)
    execs = []
    for i in range(40):
        if i % 3 == 0:
            execs.append(random_exec(rng, int(rng.integers(2, 4)), three_d=bool(i % 2)))
        elif i % 3 == 1:
            execs.append(chain((int(rng.integers(1, 200)), 1, 1), [[3, 4, 5, 3], [9, 3]], grid=(int(rng.integers(1, 4)), 1, 1)))
        else:
            execs.append(chain((int(rng.integers(1, 70)), 2, 1), [[1, 2, 1]]))
    check(ctx, port, pack(execs), len(execs))


def test_flat_path_corner_batches(ctx, port):
    """Batches the flat queue has nothing to do for: no launch at all; every exec left to the per-exec
    kernel (differing geometries); threads without events only; an exec larger than the scratch cap."""
    none = [(np.zeros((0, 6), np.uint32), [0], []) for _ in range(3)]
    check(ctx, port, pack(none), 3)
    mixed = []
    for g in range(5):
        d = np.array([[1, 1, 1, 8 + g, 1, 1], [2, 1, 1, 4, 2, 1]], np.uint32)
        ev, sites = [0], []
        for t in range(8 + g + 16):
            sites.extend([3 + (t % 3), 9, 3 + (t % 3)])
            ev.append(len(sites))
        mixed.append((d, ev, sites))
    check(ctx, port, pack(mixed), len(mixed))
    idle = [(np.array([[2, 1, 1, 70, 1, 1]] * 3, np.uint32), np.zeros(421, np.uint64), [])]
    check(ctx, port, pack(idle), 1)
    ctx.set_option("edge_scratch_mb", 1)
    try:
        big = chain((256, 1, 1), [[5, 6, 7, 5] * 10] * 4, grid=(8, 1, 1))   # 327,680 events > 262,144
        check(ctx, port, pack([big, chain((40, 1, 1), [[1, 2]]), big]), 3)
    finally:
        ctx.set_option("edge_scratch_mb", 2048)


def test_flat_path_refuses_bad_launch_offsets(ctx, edge_path):
    """launch_off that is not a CSR over the launches given is refused (HFZ_EINVAL), not read past."""
    if edge_path != "flat":
        pytest.skip("flat path only")
    tr = pack([chain((8, 1, 1), [[1, 2]]), chain((8, 1, 1), [[3]])])
    tr["launch_off"] = np.array([0, 5, 2], np.uint64)
    lo, dims, to, eo, sites = to_dev(ctx, tr)
    with pytest.raises(Exception, match="launch_off"):
        ctx.edge_record_batch(lo, dims, to, eo, sites, 2)
    ctx.synchronize()


def test_large_map_262144_edges(port, edge_path):
    """262,144-slot map: the 131,072 device counters do not fit shared memory at once -> the count kernel
    takes them in ranges (flat path) / hashed dirty-slot table (per-exec kernel)."""
    S2 = 262144
    c2 = hfz.Context(0, S2)
    c2.set_option("edge_flat", 1 if edge_path == "flat" else 0)
    try:
        tr = synth.bb_traces(3, seed=5, grid=(4, 1, 1), block=(128, 1, 1), n_launch=2)
        check(c2, port, tr, 3, S_=S2)
    finally:
        c2.close()


def test_large_map_many_distinct_slots(port, edge_path):
    """262,144-slot map, execs that touch more distinct slots than the count kernel's dirty-slot table
    holds (6,144): the exec is redone in counter passes; next to execs that stay in the table."""
    S2 = 262144
    c2 = hfz.Context(0, S2)
    c2.set_option("edge_flat", 1 if edge_path == "flat" else 0)
    try:
        rng = np.random.default_rng(29)
        execs = []
        for ex in range(4):
            dims = np.array([[4, 1, 1, 64, 1, 1]], np.uint32)
            ev, sites = [0], []
            for t in range(256):
                n = 60 if ex % 2 == 0 else 3
                sites.extend(rng.integers(0, 2 ** 32, n, dtype=np.uint64).tolist())
                ev.append(len(sites))
            execs.append((dims, ev, sites))
        check(c2, port, pack(execs), len(execs), S_=S2)
    finally:
        c2.close()


@pytest.mark.parametrize("S_", [65536, 262144])
def test_lists_output_chains_into_the_sparse_fold(port, edge_path, S_):
    """hfz_edge_record_batch_lists: the lists describe exactly the device halves the dense call writes
    (slot for slot, count for count; logical indices), an exec with more distinct slots than the list holds
    is reported as not listed, and folding the lists (hfz_feedback_batch_sparse, entry_off = e * cap) gives
    the Admit codes, signatures, virgin map and counters of folding the dense records."""
    if edge_path != "flat":
        pytest.skip("flat path only")
    c = hfz.Context(0, S_)
    H_ = S_ // 2
    try:
        rng = np.random.default_rng(37)
        tr = synth.bb_traces(24, seed=33, grid=(4, 1, 1), block=(96, 1, 1), n_launch=3)
        lo, dims, to, eo, sites = to_dev(c, tr)
        raw, ev = c.edge_record_batch(lo, dims, to, eo, sites, 24)
        raw2 = torch.zeros_like(raw)
        o = c.edge_record_batch_lists(lo, dims, to, eo, sites, 24, cap=4096, raw=raw2)
        c.synchronize()
        assert torch.equal(raw, raw2) and torch.equal(ev, o["events"])
        want_raw, want_ev = port.edge_record_batch(tr["launch_off"], tr["dims"], tr["thread_off"], tr["ev_off"], tr["sites"], 24, S_)
        assert np.array_equal(raw.cpu().numpy(), want_raw)
        ent = o["entries"].cpu().numpy().view(np.uint32).reshape(24, 4096, 2)
        ns = o["n_slots"].cpu().numpy()
        dev = raw.cpu().numpy().reshape(24, synth.record_bytes(S_))[:, H_:].view(np.uint32)
        for e in range(24):
            assert ns[e] == np.count_nonzero(dev[e]), e
            got = {int(s): int(k) for s, k in ent[e, :ns[e]]}
            assert len(got) == ns[e] and not ent[e, ns[e]:].any()
            nz = np.nonzero(dev[e])[0]
            assert got == {int(H_ + s): int(dev[e][s]) for s in nz}
        # lists only (no dense record), then the list fold against the dense fold
        o2 = c.edge_record_batch_lists(lo, dims, to, eo, sites, 24, cap=4096)
        v1, c1 = c.new_virgin(), c.new_edge_counts()
        v2, c2 = c.new_virgin(), c.new_edge_counts()
        a = c.feedback_batch(raw, v1, c1)
        b = c.feedback_batch_sparse(o2["entries"], o2["entry_off"], v2, c2)
        c.synchronize()
        for k in ("admit", "sig_full", "sig_simple", "nnz"):
            assert torch.equal(a[k], b[k]), k
        assert torch.equal(v1, v2) and torch.equal(c1, c2)
        # an exec with more distinct slots than the list holds: reported, its list stays padding
        dims1 = np.array([[4, 1, 1, 64, 1, 1]], np.uint32)
        evs, ss = [0], []
        for t in range(256):
            ss.extend(rng.integers(0, 2 ** 32, 30, dtype=np.uint64).tolist())
            evs.append(len(ss))
        tr2 = pack([(dims1, evs, ss), chain((16, 1, 1), [[1, 2, 3]])])
        lo, dims, to, eo, sites = to_dev(c, tr2)
        o3 = c.edge_record_batch_lists(lo, dims, to, eo, sites, 2, cap=4096)
        c.synchronize()
        ns3 = o3["n_slots"].cpu().numpy()
        assert ns3[0] == -1 and ns3[1] > 0
        assert not o3["entries"].cpu().numpy().reshape(2, 4096, 2)[0].any()
    finally:
        c.close()


def test_host_edge_record(ctx, port):
    rng = np.random.default_rng(13)
    seqs = [rng.integers(0, H, int(rng.integers(0, 4000)), dtype=np.uint64).astype(np.uint16) for _ in range(20)]
    seqs.append(np.zeros(3000, np.uint16))          # one slot hit 3000 times: never-zero wrap
    seqs.append(np.zeros(0, np.uint16))
    off = np.zeros(len(seqs) + 1, np.uint64)
    np.cumsum([len(s) for s in seqs], out=off[1:])
    flat = np.concatenate(seqs + [np.zeros(1, np.uint16)])
    raw = ctx.host_edge_record_batch(torch.from_numpy(off.view(np.int64)).to(ctx.device),
                                     torch.from_numpy(flat.view(np.int16)).to(ctx.device), len(seqs))
    ctx.synchronize()
    raw = raw.cpu().numpy().reshape(len(seqs), synth.record_bytes(S))
    for i, s in enumerate(seqs):
        want, _ = port.host_edge_record(s)
        assert np.array_equal(raw[i, :H], want), i
    assert raw[-2, 0] == (3000 - 1) % 255 + 1
