"""SURVEY.md 8(f) "next" rows on the GPU: f1 signature seen-sets + dispatch flags,
f2 serial-stream havoc (one Rng threaded through a block of mutants)."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import api, synth

pytestmark = pytest.mark.gpu


def seen_oracle(known: set, sigs):
    """std::set::count() then insert(), in exec order (src/engine.cpp:474-478)."""
    out = []
    for s in sigs:
        out.append(1 if s in known else 0)
        known.add(s)
    return out


def test_sigset_count_then_insert_semantics(ctx):
    rng = np.random.default_rng(1)
    s = hfz.SigSet(ctx, 1 << 16)
    known = set()
    # heavy duplication inside and across batches, plus the keys that collide with the markers
    pool = rng.integers(0, 2 ** 63, 3000, dtype=np.uint64)
    pool[0] = 0
    pool[1] = 0x9E3779B97F4A7C15
    pool[2] = (1 << 64) - 1
    for b in range(6):
        sigs = pool[rng.integers(0, 500 * (b + 1), 4000)]
        d = torch.from_numpy(sigs.view(np.int64)).to(ctx.device)
        got = s.seen_insert(d).cpu().numpy().tolist()
        assert got == seen_oracle(known, sigs.tolist()), f"batch {b}"
        assert len(s) == len(known)
    s.close()


def test_sigset_capacity_is_enforced(ctx):
    s = hfz.SigSet(ctx, 1024)
    d = torch.arange(600, dtype=torch.int64, device=ctx.device)
    s.seen_insert(d)
    with pytest.raises(hfz.HfzError) as ei:
        s.seen_insert(d + 10000)
    assert ei.value.code == 4
    s.close()


@pytest.mark.parametrize("strategy", ["all-trace", "unique-trace", "simple-trace", "coverage-increase"])
def test_dispatch_matches_run_one(ctx, checker, strategy):
    """Feedback + seen-sets + should_sanitize for two consecutive batches equals the per-exec
    sequence of Campaign::run_one (src/engine.cpp:471-478,496-498)."""
    S = 65536
    full, simple = hfz.SigSet(ctx, 1 << 16), hfz.SigSet(ctx, 1 << 16)
    virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
    v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    kf, ks = set(), set()
    for b in range(2):
        raw = synth.maps_campaign(300, S, seed=77, first=300 * b, p_extra=8, p_rare=8)
        # duplicate some maps so signatures repeat inside the batch
        rec = synth.record_bytes(S)
        raw = np.concatenate([raw, raw[: 40 * rec]])
        n = 340
        o = ctx.feedback_batch(torch.from_numpy(raw).to(ctx.device), virgin, counts)
        fs, ss, sz = hfz.dispatch_batch(ctx, full, simple, o["sig_full"], o["sig_simple"], o["admit"], strategy)
        want = checker.feedback_batch(raw, n, S, v, c)
        wf = seen_oracle(kf, want["sig_full"].tolist())
        ws = seen_oracle(ks, want["sig_simple"].tolist())
        assert fs.cpu().numpy().tolist() == wf and ss.cpu().numpy().tolist() == ws
        adm = want["admit"].tolist()
        wz = [1 if (strategy == "all-trace" or (strategy == "unique-trace" and not f) or
                    (strategy == "simple-trace" and not s_) or (strategy == "coverage-increase" and a != 0)) else 0
              for a, f, s_ in zip(adm, wf, ws)]
        assert sz.cpu().numpy().tolist() == wz
    full.close()
    simple.close()


def test_should_sanitize_truth_table(ctx):
    """tests/test_sanitizers.cpp:342-365."""
    rows = [(0, 0, 0, 1, 1, 1, 0), (0, 1, 1, 1, 0, 0, 0), (0, 0, 1, 1, 1, 0, 0), (1, 0, 0, 1, 1, 1, 1),
            (2, 0, 0, 1, 1, 1, 1), (2, 0, 1, 1, 1, 0, 1)]
    from paper_2603_12485_b200._lib import lib, check
    import ctypes as C
    # drive the flags directly through a pair of sets primed to give the wanted seen bits
    for admit, f_seen, s_seen, at, ut, st, ci in rows:
        full, simple = hfz.SigSet(ctx, 1024), hfz.SigSet(ctx, 1024)
        one = torch.tensor([5], dtype=torch.int64, device=ctx.device)
        if f_seen:
            full.seen_insert(one)
        if s_seen:
            simple.seen_insert(one)
        a = torch.tensor([admit], dtype=torch.uint8, device=ctx.device)
        for name, want in (("all-trace", at), ("unique-trace", ut), ("simple-trace", st), ("coverage-increase", ci)):
            f2, s2 = hfz.SigSet(ctx, 1024), hfz.SigSet(ctx, 1024)
            if f_seen:
                f2.seen_insert(one)
            if s_seen:
                s2.seen_insert(one)
            _, _, sz = hfz.dispatch_batch(ctx, f2, s2, one, one, a, name)
            assert int(sz[0]) == want, (admit, f_seen, s_seen, name)
            f2.close()
            s2.close()
        full.close()
        simple.close()


def test_serial_stream_havoc_block(ctx, checker):
    """One Rng threaded through 48 havoc mutants of one entry (src/engine.cpp:561-562): the
    device plan + batched kernel reproduce the serial stream byte for byte."""
    rng = np.random.default_rng(9)
    for ln, stream0 in ((300, 12345), (0, 7), (3, 99), (2500, 2 ** 63 + 11)):
        entry = rng.integers(0, 256, ln, dtype=np.uint8).tobytes()
        n = 48
        inputs = [entry] * n
        off = np.arange(n + 1, dtype=np.int64) * ln
        blob = np.frombuffer(entry * n + bytes(16), np.uint8).copy()
        d_in = torch.from_numpy(blob).to(ctx.device)
        d_off = torch.from_numpy(off).to(ctx.device)
        stream = torch.from_numpy(api.u64_to_i64(np.array([stream0], np.uint64))).to(ctx.device)
        states = ctx.havoc_serial_plan(d_off, stream)
        ob, oo, ol, dr = ctx.havoc_batch(d_in, d_off, states)
        ctx.synchronize()
        ob, oo, ol = ob.cpu().numpy(), oo.cpu().numpy(), ol.cpu().numpy()
        st = stream0
        for j in range(n):
            want, st, _ = checker.havoc(entry, st)
            assert ob[oo[j]:oo[j] + ol[j]].tobytes() == want, (ln, j)
        assert int(api.i64_to_u64(stream)[0]) == st


def test_nccl_allgather_resolve_through_the_c_abi(ctx, checker):
    """hfz_feedback_resolve_allgather (what a C/C++ host calls at N > 1): a real ncclAllGather on a
    single-rank communicator built from torch's bundled libnccl, then the rank-ordered resolve."""
    import ctypes as C
    import glob
    import os
    from paper_2603_12485_b200._lib import check, lib
    base = os.path.dirname(os.path.dirname(torch.__file__))
    cands = glob.glob(os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so*")) + glob.glob("/usr/lib/x86_64-linux-gnu/libnccl.so*")
    if not cands:
        pytest.skip("no libnccl found")
    nccl = C.CDLL(cands[0], mode=C.RTLD_GLOBAL)

    class UniqueId(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
    torch.cuda.set_device(0)
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        S, n = 65536, 300
        raw = synth.maps_campaign(n, S, seed=123, p_extra=8, p_rare=8)
        d_raw = torch.from_numpy(raw).to(ctx.device)
        virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
        scan = ctx.feedback_scan(d_raw, virgin)
        scratch = torch.empty(S, dtype=torch.uint8, device=ctx.device)
        admit = torch.empty(n, dtype=torch.uint8, device=ctx.device)
        p = lambda t: C.c_void_p(t.data_ptr())
        check(lib.hfz_feedback_resolve_allgather(ctx._h, comm, p(d_raw), n, p(virgin), p(counts), p(scan["delta"]),
                                                 p(scratch), 1, 0, p(admit)))
        ctx.synchronize()
        v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
        want = checker.feedback_batch(raw, n, S, v, c)
        assert np.array_equal(admit.cpu().numpy(), want["admit"])
        assert np.array_equal(virgin.cpu().numpy(), v) and np.array_equal(counts.cpu().numpy().view(np.uint64), c)
        assert np.array_equal(scratch.cpu().numpy(), scan["delta"].cpu().numpy())
    finally:
        nccl.ncclCommDestroy.argtypes = [C.c_void_p]
        nccl.ncclCommDestroy(comm)
