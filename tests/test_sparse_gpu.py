"""Sparse ingest parity: per-exec touched-slot lists through hfz_feedback_batch_sparse{,_host}
must give exactly what the CPU oracle gives on the dense maps the lists describe (classed
bytes, Admit codes in order, both signatures, nnz, final virgin, edge counters)."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth
from paper_2603_12485_b200._lib import HFZ_EINVAL, HfzError

pytestmark = pytest.mark.gpu

S = 65536


def cpu(checker, raw, n, S_=S, want_classed=True):
    v = np.zeros(S_, np.uint8)
    c = np.zeros(2, np.uint64)
    return checker.feedback_batch(raw, n, S_, v, c, want_classed=want_classed), v, c


def check_host(c, got, gv, gc, want):
    wo, wv, wc = want
    for k in wo:
        assert np.array_equal(got[k], wo[k]), f"{k} differs at {np.nonzero(got[k] != wo[k])[0][:8]}"
    assert np.array_equal(gv, wv), "virgin differs"
    assert np.array_equal(gc, wc), f"edge counts differ {gc} vs {wc}"


@pytest.fixture(params=["native", "expand"])
def sctx(request):
    """Own context per test (the sparse chunk size can only be set before first use); every test
    runs through both device paths: rank + chain kernels on the lists, and expansion into dense
    staging records scanned by K2."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = hfz.Context(0)
    c.set_option("sparse_native", 1 if request.param == "native" else 0)
    yield c
    c.close()


@pytest.mark.parametrize("mode,shuffle", [("campaign", 1), ("iid", 7), ("campaign", None)])
def test_sparse_host_equals_oracle(sctx, checker, mode, shuffle):
    n = 700
    raw = synth.maps_iid(n, S) if mode == "iid" else synth.maps_campaign(n, S, p_extra=16, p_rare=16)
    entries, off = synth.to_sparse(raw, n, S, shuffle_seed=shuffle)
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    got = sctx.feedback_batch_sparse_host(entries, off, v, c, want_classed=True)
    check_host(sctx, got, v, c, cpu(checker, raw, n))
    assert len(set(got["admit"].tolist())) >= 2


def test_sparse_chunking_and_reuse(sctx, checker):
    """Several chunks per call (chunk = 64 execs), the staging buffer must come back all-zero:
    a second, different batch through the same context must still be exact."""
    sctx.set_option("sparse_chunk", 64)
    for seed, n in ((5, 333), (6, 190), (7, 64), (8, 1)):
        raw = synth.maps_campaign(n, S, seed=seed, p_extra=8, p_rare=8)
        entries, off = synth.to_sparse(raw, n, S, shuffle_seed=seed)
        v = np.zeros(S, np.uint8)
        c = np.zeros(2, np.uint64)
        got = sctx.feedback_batch_sparse_host(entries, off, v, c, want_classed=True)
        check_host(sctx, got, v, c, cpu(checker, raw, n))


def test_sparse_edge_vectors_and_empty_execs(sctx, checker):
    """All-zero map (empty list), full-density map, rung boundaries, last/first slots; plus
    explicit count-0 pairs, which must read as unvisited."""
    raw, n = synth.maps_edge_cases(S)
    entries, off = synth.to_sparse(raw, n, S)
    assert off[1] == 0  # the all-zero map has an empty list
    # append two count-0 pairs to the last exec
    entries = np.concatenate([entries, np.array([[77, 0], [S - 5, 0]], np.uint32)])
    off = off.copy()
    off[-1] += 2
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    got = sctx.feedback_batch_sparse_host(entries, off, v, c, want_classed=True)
    check_host(sctx, got, v, c, cpu(checker, raw, n))


def test_sparse_device_call_equals_dense_call(sctx):
    """Device-buffer form against the dense device call, with a pre-warmed virgin map."""
    n = 300
    warm = synth.maps_campaign(256, S, seed=90)
    raw = synth.maps_campaign(n, S, seed=91, p_extra=8, p_rare=8)
    dev = sctx.device
    results = []
    for sparse in (False, True):
        virgin, counts = sctx.new_virgin(), sctx.new_edge_counts()
        sctx.feedback_batch(torch.from_numpy(warm).to(dev), virgin, counts)
        if sparse:
            entries, off = synth.to_sparse(raw, n, S, shuffle_seed=3)
            o = sctx.feedback_batch_sparse(torch.from_numpy(entries.view(np.int32)).to(dev),
                                           torch.from_numpy(off.view(np.int64)).to(dev), virgin, counts,
                                           want_classed=True)
        else:
            o = sctx.feedback_batch(torch.from_numpy(raw).to(dev), virgin, counts, want_classed=True)
        sctx.synchronize()
        results.append({k: t.cpu().numpy() for k, t in o.items()} | {"virgin": virgin.cpu().numpy(),
                                                                      "counts": counts.cpu().numpy()})
    for k in results[0]:
        assert np.array_equal(results[0][k], results[1][k]), k


def test_expand_sparse_reproduces_records(sctx):
    n = 100
    raw = synth.maps_iid(n, S, seed=11)
    entries, off = synth.to_sparse(raw, n, S, shuffle_seed=2)
    out = sctx.expand_sparse(torch.from_numpy(entries.view(np.int32)).to(sctx.device),
                             torch.from_numpy(off.view(np.int64)).to(sctx.device))
    sctx.synchronize()
    assert np.array_equal(out.cpu().numpy(), raw)


def test_sparse_out_of_range_pairs_are_reported(sctx, checker):
    """Pairs naming a slot >= S are ignored, the fold completes, and the host call says so."""
    n = 40
    raw = synth.maps_campaign(n, S, seed=21)
    entries, off = synth.to_sparse(raw, n, S)
    bad = np.concatenate([entries, np.array([[S, 3], [0xFFFFFFFF, 1]], np.uint32)])
    off2 = off.copy()
    off2[-1] += 2
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    with pytest.raises(HfzError) as ei:
        sctx.feedback_batch_sparse_host(bad, off2, v, c)
    assert ei.value.code == HFZ_EINVAL
    wo, wv, wc = cpu(checker, raw, n, want_classed=False)
    assert np.array_equal(v, wv) and np.array_equal(c, wc)
    # and the context is still usable and exact afterwards
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    got = sctx.feedback_batch_sparse_host(entries, off, v, c)
    assert np.array_equal(got["admit"], wo["admit"]) and np.array_equal(got["sig_full"], wo["sig_full"])


def test_sparse_bad_offsets_rejected(sctx):
    entries = np.zeros((4, 2), np.uint32)
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    with pytest.raises(HfzError):
        sctx.feedback_batch_sparse_host(entries, np.array([0, 3, 2], np.uint64), v, c)


def test_sparse_subrange_folds_equal_one_fold(sctx, checker):
    """entry_off indexes the pairs absolutely: folding execs [0,k) and then [k,n) through
    entry_off[k:] (entry_off[0] != 0) equals one fold of the whole batch."""
    n, k = 150, 61
    raw = synth.maps_campaign(n, S, seed=41, p_extra=8, p_rare=8)
    entries, off = synth.to_sparse(raw, n, S, shuffle_seed=9)
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    a = sctx.feedback_batch_sparse_host(entries, off[:k + 1].copy(), v, c)
    b = sctx.feedback_batch_sparse_host(entries, off[k:].copy(), v, c)
    wo, wv, wc = cpu(checker, raw, n, want_classed=False)
    for key in wo:
        assert np.array_equal(np.concatenate([a[key], b[key]]), wo[key]), key
    assert np.array_equal(v, wv) and np.array_equal(c, wc)


@pytest.mark.parametrize("S2,native,n", [(262144, 1, 48), (262144, 0, 48), (1 << 20, 1, 5)])
def test_sparse_large_map(S2, native, n):
    """262,144-slot map (BASELINE.json configs[2]) through the list-native kernels (4 warps per CTA:
    a 32 KB bitmap each) and through the dense-staging fallback; 2^20 slots, the largest map whose
    bitmap fits one warp's shared memory."""
    from oracle import pyoracle
    checker_large = pyoracle.best_checker(S2)
    c2 = hfz.Context(0, S2)
    c2.set_option("sparse_native", native)
    try:
        raw = synth.maps_iid(n, S2, seed=31)
        entries, off = synth.to_sparse(raw, n, S2, shuffle_seed=4)
        v = np.zeros(S2, np.uint8)
        c = np.zeros(2, np.uint64)
        got = c2.feedback_batch_sparse_host(entries, off, v, c)
        wo, wv, wc = cpu(checker_large, raw, n, S2, want_classed=False)
        for k in wo:
            assert np.array_equal(got[k], wo[k]), k
        assert np.array_equal(v, wv) and np.array_equal(c, wc)
    finally:
        c2.close()


def test_sparse_repeated_pairs_with_equal_counts(sctx, checker):
    """A slot listed twice with the same count (SparseBatch does that after device_store(x, 0)
    followed by a new store) is one slot: nnz, signatures and virgin are those of the map."""
    n = 60
    raw = synth.maps_campaign(n, S, seed=55, p_extra=8, p_rare=8)
    entries, off = synth.to_sparse(raw, n, S, shuffle_seed=6)
    parts, new_off = [], [0]
    for e in range(n):
        seg = entries[int(off[e]):int(off[e + 1])]
        dup = seg[:: 7]                                   # every 7th pair once more
        parts += [seg, dup]
        new_off.append(new_off[-1] + len(seg) + len(dup))
    entries2 = np.ascontiguousarray(np.concatenate(parts))
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    got = sctx.feedback_batch_sparse_host(entries2, np.array(new_off, np.uint64), v, c, want_classed=True)
    check_host(sctx, got, v, c, cpu(checker, raw, n))


@pytest.mark.parametrize("S_small", [1024, 4096, 32768])
@pytest.mark.parametrize("native", [1, 0])
def test_small_map_sizes(port, S_small, native):
    """Map sizes below the reference's 65,536 (run-time parameter of the C restatement): the
    bitmap / prefix geometry of the rank kernel and the dense kernels' row walk must adapt."""
    c2 = hfz.Context(0, S_small)
    c2.set_option("sparse_native", native)
    try:
        n = 90
        raw = synth.maps_iid(n, S_small, density=0.05, seed=61)
        entries, off = synth.to_sparse(raw, n, S_small, shuffle_seed=8)
        v, c = np.zeros(S_small, np.uint8), np.zeros(2, np.uint64)
        got = c2.feedback_batch_sparse_host(entries, off, v, c, want_classed=True)
        wv, wc = np.zeros(S_small, np.uint8), np.zeros(2, np.uint64)
        want = port.feedback_batch(raw, n, S_small, wv, wc, want_classed=True)
        for k in want:
            assert np.array_equal(got[k], want[k]), k
        assert np.array_equal(v, wv) and np.array_equal(c, wc)
        # and the dense host path on the same maps
        v2, c3 = np.zeros(S_small, np.uint8), np.zeros(2, np.uint64)
        got2 = c2.feedback_batch_host(raw, v2, c3)
        assert np.array_equal(got2["admit"], want["admit"]) and np.array_equal(got2["sig_full"], want["sig_full"])
        assert np.array_equal(v2, wv)
    finally:
        c2.close()


def test_sparse_empty_batch_and_all_empty_lists(sctx):
    v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    got = sctx.feedback_batch_sparse_host(np.zeros((0, 2), np.uint32), np.zeros(1, np.uint64), v, c)
    assert got["admit"].size == 0 and not v.any()
    got = sctx.feedback_batch_sparse_host(np.zeros((0, 2), np.uint32), np.zeros(6, np.uint64), v, c)
    assert got["admit"].tolist() == [0] * 5 and got["nnz"].tolist() == [0] * 5
    assert all(int(x) == 14695981039346656037 for x in got["sig_full"]) and not v.any() and not c.any()


@pytest.mark.parametrize("mode", ["campaign", "iid", "edge"])
def test_compact_lists_equal_oracle(checker, mode):
    """The 4-byte list form (slot | count << 16, wide pairs for counts >= 65,536)."""
    c = hfz.Context(0)
    try:
        if mode == "edge":
            raw, n = synth.maps_edge_cases(S)
        else:
            n = 500
            raw = synth.maps_iid(n, S, seed=71) if mode == "iid" else synth.maps_campaign(n, S, seed=72, p_extra=8, p_rare=8)
        compact, coff, wide, woff = synth.to_compact(raw, n, S, shuffle_seed=11)
        assert wide.shape[0] > 0  # device counts of 65,536 and more occur in every mode
        v, cnt = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        got = c.feedback_batch_compact_host(compact, coff, wide, woff, v, cnt, want_classed=True)
        check_host(c, got, v, cnt, cpu(checker, raw, n))
        # sub-range folds through absolute offsets, compact list only when an exec has no wide pairs
        v2, cnt2 = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        k = n // 3
        a = c.feedback_batch_compact_host(compact, coff[:k + 1].copy(), wide, woff[:k + 1].copy(), v2, cnt2)
        b = c.feedback_batch_compact_host(compact, coff[k:].copy(), wide, woff[k:].copy(), v2, cnt2)
        assert np.array_equal(np.concatenate([a["admit"], b["admit"]]), got["admit"])
        assert np.array_equal(np.concatenate([a["sig_full"], b["sig_full"]]), got["sig_full"])
        assert np.array_equal(v2, v) and np.array_equal(cnt2, cnt)
    finally:
        c.close()


@pytest.mark.parametrize("mode", ["campaign", "iid", "edge"])
def test_packed_lists_equal_oracle(checker, mode):
    """The packed form: 3-byte host-half entries (every exec padded to a multiple of four), 4-byte device-half
    entries with the count clipped at 65,536 (the last rung's lower bound: every class survives the clip)."""
    c = hfz.Context(0)
    try:
        if mode == "edge":
            raw, n = synth.maps_edge_cases(S)
        else:
            n = 5000 if mode == "campaign" else 500  # 5,000 execs: two chunks of the H2D stream
            raw = synth.maps_iid(n, S, seed=81) if mode == "iid" else synth.maps_campaign(n, S, seed=82, p_extra=8, p_rare=8)
        h3, hoff, d17, doff = synth.to_packed(raw, n, S, shuffle_seed=13)
        assert int((d17 >> 15).max()) == 65536 and (hoff % 4 == 0).all()
        v, cnt = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        want_classed = n <= 1000
        got = c.feedback_batch_packed_host(h3, hoff, d17, doff, v, cnt, want_classed=want_classed)
        if want_classed:
            check_host(c, got, v, cnt, cpu(checker, raw, n))
        else:
            wo, wv, wc = cpu(checker, raw, n, want_classed=False)
            for key in wo:
                assert np.array_equal(got[key], wo[key]), key
            assert np.array_equal(v, wv) and np.array_equal(cnt, wc)
        # sub-range folds through absolute offsets
        v2, cnt2 = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        k = n // 3
        a = c.feedback_batch_packed_host(h3, hoff[:k + 1].copy(), d17, doff[:k + 1].copy(), v2, cnt2)
        b = c.feedback_batch_packed_host(h3, hoff[k:].copy(), d17, doff[k:].copy(), v2, cnt2)
        assert np.array_equal(np.concatenate([a["admit"], b["admit"]]), got["admit"])
        assert np.array_equal(np.concatenate([a["sig_full"], b["sig_full"]]), got["sig_full"])
        assert np.array_equal(v2, v) and np.array_equal(cnt2, cnt)
    finally:
        c.close()


def test_packed_lists_corner_cases_and_rejections(checker):
    c = hfz.Context(0)
    try:
        H = S // 2
        v, cnt = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        # exec 0: nothing; exec 1: host slots only (5 entries + 3 padding); exec 2: device slots only, one of
        # them listed with count 0 (ignored); exec 3: the last slot of each half
        h3 = np.zeros((12, 3), np.uint8)
        for i, (slot, count) in enumerate([(7, 1), (300, 255), (32767, 9), (256, 4), (1, 128)]):
            h3[i] = (slot & 0xFF, slot >> 8, count)
        h3[8] = (0xFF, 0x7F, 3)  # exec 3: slot 32767
        hoff = np.array([0, 0, 8, 8, 12], np.uint64)
        d17 = np.array([5 | 65536 << 15, 9 | 0 << 15, 10 | 2 << 15, 32767 | 600 << 15], np.uint32)  # 70,000 clipped to 65,536
        doff = np.array([0, 0, 0, 3, 4], np.uint64)
        raw = np.zeros((4, 5 * H), np.uint8)
        for slot, count in [(7, 1), (300, 255), (32767, 9), (256, 4), (1, 128)]:
            raw[1, slot] = count
        dev = raw[:, H:].view(np.uint32)
        dev[2, 5] = 70000
        dev[2, 10] = 2
        raw[3, 32767] = 3
        dev[3, 32767] = 600
        got = c.feedback_batch_packed_host(np.ascontiguousarray(h3.reshape(-1)), hoff, d17, doff, v, cnt, want_classed=True)
        check_host(c, got, v, cnt, cpu(checker, np.ascontiguousarray(raw.reshape(-1)), 4))
        assert got["nnz"].tolist() == [0, 5, 2, 2]
        with pytest.raises(HfzError):  # an exec's host list that is not padded to four entries
            c.feedback_batch_packed_host(np.ascontiguousarray(h3.reshape(-1)), np.array([0, 5, 8, 8, 12], np.uint64), d17, doff, v, cnt)
        with pytest.raises(HfzError):  # decreasing offsets
            c.feedback_batch_packed_host(np.ascontiguousarray(h3.reshape(-1)), hoff, d17, np.array([0, 3, 0, 3, 4], np.uint64), v, cnt)
        c2 = hfz.Context(0, 262144)
        try:
            with pytest.raises(HfzError):  # 15-bit slots per half: the 65,536-slot map only
                c2.feedback_batch_packed_host(np.ascontiguousarray(h3.reshape(-1)), hoff, d17, doff,
                                              np.zeros(262144, np.uint8), np.zeros(2, np.uint64))
        finally:
            c2.close()
    finally:
        c.close()


def test_compact_without_wide_list_and_rejections(checker):
    c = hfz.Context(0)
    try:
        n = 64
        raw = synth.maps_campaign(n, S, seed=73)
        H = S // 2
        recs = raw.reshape(n, -1)
        dev = recs[:, H:].view(np.uint32)
        dev[dev >= 65536] = 65535                      # no wide pairs needed
        compact, coff, wide, woff = synth.to_compact(raw, n, S)
        assert wide.shape[0] == 0
        v, cnt = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        got = c.feedback_batch_compact_host(compact, coff, None, None, v, cnt)
        wo, wv, wc = cpu(checker, raw, n, want_classed=False)
        for key in wo:
            assert np.array_equal(got[key], wo[key]), key
        assert np.array_equal(v, wv) and np.array_equal(cnt, wc)
        c.set_option("sparse_native", 0)               # the expand fallback has no compact form
        with pytest.raises(HfzError):
            c.feedback_batch_compact_host(compact, coff, None, None, v, cnt)
    finally:
        c.close()


def test_calls_on_a_non_default_stream(checker):
    """Everything is enqueued on the context's stream (here a non-default torch stream): dense,
    sparse and compact folds interleaved with torch work on the same stream stay ordered."""
    c = hfz.Context(0)
    try:
        n = 200
        raw = synth.maps_campaign(n, S, seed=81, p_extra=8, p_rare=8)
        wo, wv, wc = cpu(checker, raw, n, want_classed=False)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            d_raw = torch.from_numpy(raw).to(c.device, non_blocking=True)
            virgin, counts = c.new_virgin(), c.new_edge_counts()
            o = c.feedback_batch(d_raw, virgin, counts)
            admit_sum = o["admit"].sum()              # torch op queued behind the fold on the same stream
            entries, off = synth.to_sparse(raw, n, S, shuffle_seed=5)
            d_ent = torch.from_numpy(entries.view(np.int32)).to(c.device, non_blocking=True)
            d_off = torch.from_numpy(off.view(np.int64)).to(c.device, non_blocking=True)
            v2, c2 = c.new_virgin(), c.new_edge_counts()
            o2 = c.feedback_batch_sparse(d_ent, d_off, v2, c2)
        s.synchronize()
        assert int(admit_sum) == int(wo["admit"].sum())
        assert np.array_equal(o["admit"].cpu().numpy(), wo["admit"]) and np.array_equal(virgin.cpu().numpy(), wv)
        assert np.array_equal(o2["sig_full"].cpu().numpy().view(np.uint64), wo["sig_full"])
        assert np.array_equal(v2.cpu().numpy(), wv) and np.array_equal(c2.cpu().numpy().view(np.uint64), wc)
        with torch.cuda.stream(s):
            vh, ch = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
            comp, coff, wide, woff = synth.to_compact(raw, n, S)
            o3 = c.feedback_batch_compact_host(comp, coff, wide, woff, vh, ch)
        assert np.array_equal(o3["admit"], wo["admit"]) and np.array_equal(vh, wv)
    finally:
        c.close()
