"""K2/K2b/K4 parity: the CUDA feedback path vs the CPU oracle, bit-exact, through the C-ABI.

Compared per exec: classed map bytes, Admit code, Full and Simple signatures, nnz; after the
batch: every virgin byte and both distinct-edge counters.
"""
import numpy as np
import pytest
import torch

from paper_2603_12485_b200 import synth

pytestmark = pytest.mark.gpu

S = 65536


KERNEL_OPTS = {  # (scan_small, scan_pipe, scan_two_stage, small_fused): force one of the five dense paths
    "lane_per_map": (0, 0, 0, 0),
    "warp_per_map": (1 << 40, 0, 0, 0),
    "pipelined": (0, 1 << 20, 0, 0),
    "two_stage": (0, 0, 1 << 40, 0),
    "fused_step": (0, 0, 1 << 40, 1),   # the two-stage fold as ONE cooperative launch (the small-batch default)
}


def force_kernel(c, name):
    small, pipe, two, fused = KERNEL_OPTS[name]
    c.set_option("scan_small", small)
    c.set_option("scan_pipe", pipe)
    c.set_option("scan_two_stage", two)
    c.set_option("small_fused", fused)


@pytest.fixture(autouse=True, params=list(KERNEL_OPTS))
def scan_kernel(request, ctx):
    """Every test runs against all five dense paths: the throughput kernel (32 maps per warp),
    the warp-per-map kernel, the pipelined kernel (producer warps + one consumer warp per 32 maps),
    the two-stage path (compact + chain) and the fused step (the same fold as one cooperative
    launch); by default the library picks by batch size."""
    force_kernel(ctx, request.param)
    yield request.param
    for k in ("scan_small", "scan_pipe", "scan_two_stage"):
        ctx.set_option(k, -1)
    ctx.set_option("small_fused", 1)


def run_gpu(ctx, raw, virgin0=None, counts0=None, want_classed=True):
    d_raw = torch.from_numpy(raw).to(ctx.device)
    virgin = ctx.new_virgin() if virgin0 is None else torch.from_numpy(virgin0).to(ctx.device)
    counts = ctx.new_edge_counts() if counts0 is None else torch.from_numpy(counts0.view(np.int64)).to(ctx.device)
    o = ctx.feedback_batch(d_raw, virgin, counts, want_classed=want_classed)
    ctx.synchronize()
    res = dict(admit=o["admit"].cpu().numpy(), sig_full=o["sig_full"].cpu().numpy().view(np.uint64),
               sig_simple=o["sig_simple"].cpu().numpy().view(np.uint64),
               nnz=o["nnz"].cpu().numpy().view(np.uint32))
    if want_classed:
        res["classed"] = o["classed"].cpu().numpy()
    return res, virgin.cpu().numpy(), counts.cpu().numpy().view(np.uint64)


def run_cpu(checker, raw, n, S_=S, virgin0=None, counts0=None, want_classed=True):
    v = np.zeros(S_, np.uint8) if virgin0 is None else virgin0.copy()
    c = np.zeros(2, np.uint64) if counts0 is None else counts0.copy()
    o = checker.feedback_batch(raw, n, S_, v, c, want_classed=want_classed)
    return o, v, c


def assert_same(g, c):
    (go, gv, gc), (co, cv, cc) = g, c
    for k in co:
        assert np.array_equal(go[k], co[k]), f"{k} differs at {np.nonzero(go[k] != co[k])[0][:8]}"
    assert np.array_equal(gv, cv), "virgin differs"
    assert np.array_equal(gc, cc), f"edge counts differ {gc} vs {cc}"


@pytest.mark.parametrize("mode", ["iid", "campaign"])
def test_config1_cold_start_1024(ctx, checker, mode):
    """BASELINE.json configs[0]: 1,024 maps, ~2 % density, virgin starts empty so all three
    Admit codes occur; the whole ordered sequence is compared."""
    raw = synth.maps_iid(1024, S) if mode == "iid" else synth.maps_campaign(1024, S)
    g = run_gpu(ctx, raw)
    c = run_cpu(checker, raw, 1024)
    assert_same(g, c)
    assert len(set(c[0]["admit"].tolist())) >= 2


def test_edge_vectors(ctx, checker):
    raw, n = synth.maps_edge_cases(S)
    assert_same(run_gpu(ctx, raw), run_cpu(checker, raw, n))
    # and again in reverse order (full-density map last)
    rec = synth.record_bytes(S)
    rev = raw.reshape(n, rec)[::-1].copy().reshape(-1)
    assert_same(run_gpu(ctx, rev), run_cpu(checker, rev, n))


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 65, 257])
def test_ragged_batch_sizes(ctx, checker, n):
    raw = synth.maps_campaign(n, S, seed=1000 + n)
    assert_same(run_gpu(ctx, raw), run_cpu(checker, raw, n))


def test_empty_batch(ctx):
    virgin = ctx.new_virgin()
    counts = ctx.new_edge_counts()
    raw = torch.zeros(0, dtype=torch.uint8, device=ctx.device)
    o = ctx.feedback_batch(raw, virgin, counts)
    ctx.synchronize()
    assert o["admit"].numel() == 0 and int(virgin.sum()) == 0 and int(counts.sum()) == 0


def test_virgin_carried_across_batches(ctx, checker):
    """Warm virgin: fold 512 maps, then 512 more in a second call; equals one 1,024 fold."""
    raw = synth.maps_campaign(1024, S, seed=77)
    rec = synth.record_bytes(S)
    a, b = raw[: 512 * rec], raw[512 * rec:]
    d_v, d_c = ctx.new_virgin(), ctx.new_edge_counts()
    o1 = ctx.feedback_batch(torch.from_numpy(a).to(ctx.device), d_v, d_c)
    adm1 = o1["admit"].cpu().numpy()
    o2 = ctx.feedback_batch(torch.from_numpy(b).to(ctx.device), d_v, d_c)
    adm2 = o2["admit"].cpu().numpy()
    co, cv, cc = run_cpu(checker, raw, 1024, want_classed=False)
    assert np.array_equal(np.concatenate([adm1, adm2]), co["admit"])
    assert np.array_equal(d_v.cpu().numpy(), cv)
    assert np.array_equal(d_c.cpu().numpy().view(np.uint64), cc)


def test_reference_known_answers(ctx):
    """tests/test_coverage.cpp:157-259 restated: classify example, Admit sequence on slot
    42/43/dev+9, OR-folding, byte-level FNV values."""
    rec = synth.record_bytes(S)
    H = S // 2

    def mk(host=(), dev=()):
        r = np.zeros(rec, np.uint8)
        for i, v in host:
            r[i] = v
        d = r[H:].view(np.uint32)
        for i, v in dev:
            d[i - H] = v
        return r

    # signatures: {5: 3 hits -> class 4, 40000: 700 -> class 8}
    m = mk(host=[(5, 3)], dev=[(40000, 700)])
    (o, _, _) = run_gpu(ctx, m)
    assert int(o["sig_simple"][0]) == 0x2E1A3655EF7B3874
    assert int(o["sig_full"][0]) == 0x31CF681E15834C40
    assert o["classed"][0][5] == 4 and o["classed"][0][40000] == 8 and o["nnz"][0] == 2
    (o, _, _) = run_gpu(ctx, mk())
    assert int(o["sig_simple"][0]) == 0xCBF29CE484222325 == int(o["sig_full"][0])
    # classify example (test_coverage.cpp:157-175)
    (o, _, _) = run_gpu(ctx, mk(host=[(10, 1), (500, 5)], dev=[(H + 3, 700), (S - 1, 2)]))
    assert np.nonzero(o["classed"][0])[0].tolist() == [10, 500, H + 3, S - 1]
    assert o["classed"][0][[10, 500, H + 3, S - 1]].tolist() == [1, 8, 8, 2]
    # Admit sequence (test_coverage.cpp:177-221)
    seq = [mk(host=[(42, 1)]), mk(host=[(42, 1)]), mk(host=[(42, 2)]), mk(host=[(42, 4)]),
           mk(host=[(42, 5)]), mk(host=[(42, 3), (43, 1)]), mk(dev=[(H + 9, 1)])]
    (o, v, c) = run_gpu(ctx, np.concatenate(seq))
    assert o["admit"].tolist() == [2, 0, 1, 1, 0, 2, 2]
    assert c.tolist() == [2, 1]
    # OR-folding (test_coverage.cpp:223-237)
    (o, v, c) = run_gpu(ctx, np.concatenate([mk(host=[(100, 9)], dev=[(H + 5, 600)]), mk(host=[(100, 1)])]))
    assert v[100] == (16 | 1) and v[H + 5] == 8


def test_host_buffer_path(ctx, checker):
    """hfz_feedback_batch_host: chunked H2D staging gives the same fold."""
    raw = synth.maps_campaign(300, S, seed=5)
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    o = ctx.feedback_batch_host(raw, v, c, want_classed=True)
    co, cv, cc = run_cpu(checker, raw, 300)
    for k in co:
        assert np.array_equal(o[k], co[k]), k
    assert np.array_equal(v, cv) and np.array_equal(c, cc)


def test_sharded_scan_resolve_equals_sequential(ctx, checker, scan_kernel):
    """R simulated ranks on one GPU -- per-rank scan against V0, 'allgather' of
    the deltas by concatenation, resolve in rank order -- must reproduce the single-rank
    sequential Admit codes, virgin and counters."""
    R, per = 4, 96
    rec = synth.record_bytes(S)
    warm = synth.maps_campaign(64, S, seed=9)
    raw = synth.maps_campaign(R * per, S, seed=9, first=64, p_extra=8, p_rare=8)
    v0 = np.zeros(S, np.uint8)
    c0 = np.zeros(2, np.uint64)
    checker.feedback_batch(warm, 64, S, v0, c0)
    co, cv, cc = run_cpu(checker, raw, R * per, virgin0=v0, counts0=c0, want_classed=False)
    shards = [torch.from_numpy(raw[r * per * rec:(r + 1) * per * rec]).to(ctx.device) for r in range(R)]
    d_v0 = torch.from_numpy(v0).to(ctx.device)
    import paper_2603_12485_b200 as hfz
    ctxs = [hfz.Context(0) for _ in range(R)]
    for i, c in enumerate(ctxs):
        # mix the kernels across the simulated ranks
        force_kernel(c, list(KERNEL_OPTS)[(i + list(KERNEL_OPTS).index(scan_kernel)) % len(KERNEL_OPTS)])
    try:
        scans = [ctxs[r].feedback_scan(shards[r], d_v0) for r in range(R)]
        deltas = torch.cat([s["delta"] for s in scans])
        admits, virgins, counts = [], [], []
        for r in range(R):
            v = d_v0.clone()
            c = torch.from_numpy(c0.view(np.int64).copy()).to(ctx.device)
            admits.append(ctxs[r].feedback_resolve(shards[r], v, c, deltas, R, r).cpu().numpy())
            virgins.append(v.cpu().numpy())
            counts.append(c.cpu().numpy().view(np.uint64))
        assert np.array_equal(np.concatenate(admits), co["admit"])
        for r in range(R):
            assert np.array_equal(virgins[r], cv) and np.array_equal(counts[r], cc)
        sf = np.concatenate([s["sig_full"].cpu().numpy().view(np.uint64) for s in scans])
        assert np.array_equal(sf, co["sig_full"])
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("opts", [dict(scan_row=512), dict(scan_row=256, scan_prefetch=0), dict(scan_row=512, scan_prefetch=0),
                                  dict(scan_row=512, virgin_smem=0), dict(scan_row=256, virgin_smem=0), dict(scan_row=256, scan_warps=3),
                                  dict(scan_row=1024), dict(scan_row=1024, virgin_smem=0), dict(scan_row=1024, scan_prefetch=0, scan_warps=2)])
def test_scan_tunings_agree(ctx, checker, opts):
    """Every tuning of the scan kernel (row size, warps, L2 prefetch, virgin in smem or not)
    is the same function."""
    raw = synth.maps_campaign(200, S, seed=31)
    for k, v in opts.items():
        ctx.set_option(k, v)
    try:
        assert_same(run_gpu(ctx, raw), run_cpu(checker, raw, 200))
    finally:
        for k, v in dict(scan_row=0, scan_warps=0, scan_prefetch=1, virgin_smem=1).items():
            ctx.set_option(k, v)


@pytest.mark.parametrize("n", [1, 15, 16, 17, 33, 16 * 148 * 2 + 5, 16 * 148 * 9 * 2 + 21])
def test_sixteen_maps_per_warp(ctx, checker, n, scan_kernel):
    """scan_row = 1024: a warp takes 16 maps (lanes 16..31 idle in the chain phase), for batches that leave most
    warps of the grid without a 32-map group.  Full and partial groups, one and several groups per warp."""
    if scan_kernel != "lane_per_map":
        pytest.skip("lane-per-map kernel only")
    raw = synth.maps_campaign(n, S, seed=59)
    ctx.set_option("scan_row", 1024)
    try:
        assert_same(run_gpu(ctx, raw, want_classed=n < 64), run_cpu(checker, raw, n, want_classed=n < 64))
    finally:
        ctx.set_option("scan_row", 0)


def test_many_maps_per_warp(ctx, checker):
    """More maps than one group per warp: 3 warps x 148 CTAs must walk 32+ maps each."""
    n = 148 * 3 * 32 + 148 * 3 * 5 + 7
    raw = synth.maps_campaign(n, S, seed=13)
    ctx.set_option("scan_warps", 3)
    try:
        assert_same(run_gpu(ctx, raw, want_classed=False), run_cpu(checker, raw, n, want_classed=False))
    finally:
        ctx.set_option("scan_warps", 0)


@pytest.mark.parametrize("n,mode", [(9000, "iid"), (13000, "campaign"), (20000, "iid")])
def test_every_map_novel_at_throughput_sizes(ctx, checker, n, mode, scan_kernel):
    """An empty virgin map under a batch large enough for the automatic dispatch to take the pipelined and the
    lane-per-map kernels: every map shows something new versus V0, thousands of them own an entry of the
    first-occurrence table, and the Admit codes come from the table pass alone (no candidate is walked).
    All three codes occur; iid maps keep ~a quarter of the batch admitted to the end."""
    if scan_kernel != "lane_per_map":
        pytest.skip("one pass: the dispatch is left automatic")
    for k in ("scan_small", "scan_pipe", "scan_two_stage"):
        ctx.set_option(k, -1)
    ctx.set_option("small_fused", 1)
    raw = (synth.maps_iid if mode == "iid" else synth.maps_campaign)(n, S, seed=77)
    g = run_gpu(ctx, raw, want_classed=False)
    c = run_cpu(checker, raw, n, want_classed=False)
    assert_same(g, c)
    codes = np.bincount(g[0]["admit"], minlength=3)
    assert codes[2] > 0 and codes[0] > 0 and (mode == "campaign" or codes[1] > 0)


def test_large_map_262144(checker, scan_kernel):
    """BASELINE.json configs[2] map size: 262,144 slots (virgin no longer fits shared memory)."""
    import paper_2603_12485_b200 as hfz
    from oracle import pyoracle
    S2 = 262144
    ck = pyoracle.Ref(S2) if pyoracle.Ref.available(S2) else pyoracle.Port()
    c2 = hfz.Context(0, S2)
    force_kernel(c2, scan_kernel)
    try:
        raw = synth.maps_iid(48, S2, density=0.01, seed=3)
        g = run_gpu(c2, raw)
        c = run_cpu(ck, raw, 48, S_=S2)
        assert_same(g, c)
    finally:
        c2.close()


@pytest.mark.parametrize("row", [256, 512])
@pytest.mark.parametrize("n", [32 * 148 * 2 + 13, 32 * 5, 1000])
def test_pipelined_kernel_rows_and_teams(ctx, checker, row, n, scan_kernel):
    """Medium-batch kernel with both ring-slot sizes, more groups than SMs x teams (several CTAs
    per SM in waves), a partial last group and idle teams."""
    if scan_kernel != "pipelined":
        pytest.skip("pipelined kernel only")
    raw = synth.maps_campaign(n, S, seed=77 + row, p_extra=32, p_rare=32)
    ctx.set_option("scan_row", row)
    try:
        assert_same(run_gpu(ctx, raw, want_classed=False), run_cpu(checker, raw, n, want_classed=False))
    finally:
        ctx.set_option("scan_row", 0)


def test_warp_fnv():
    """The warp-parallel FNV-1a (csrc/hfz_fnv.cuh: bit-sliced low-byte chain + affine sum) equals the
    byte-serial definition of trace_signature (src/coverage.cpp:89-97) on ordered entry lists of every
    block-boundary length; the empty list gives the offset basis (tests/test_coverage.cpp:239-259)."""
    import ctypes as C
    from paper_2603_12485_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    lib.hfz_dbg_warp_fnv.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    P, M = (1 << 40) + 0x1b3, (1 << 64) - 1

    def serial(entries, full):
        h = 0xcbf29ce484222325
        for e in entries:
            for b in ((e & 0xff, (e >> 8) & 0xff, 1 << (e >> 24)) if full else (e & 0xff, (e >> 8) & 0xff)):
                h = ((h ^ b) * P) & M
        return h

    rng = np.random.default_rng(31)
    for n in (0, 1, 2, 10, 11, 341, 342, 511, 512, 513, 682, 683, 1023, 1024, 1025, 1311, 2048, 2049, 5243):
        slots = np.sort(rng.choice(1 << 18, n, replace=False)).astype(np.uint32) if n else np.zeros(0, np.uint32)
        rung = rng.integers(0, 8, n).astype(np.uint32)
        en = np.ascontiguousarray((slots & 0xFFFFFF) | (rung << 24), np.uint32)
        out = np.zeros(2, np.uint64)
        src = en if n else np.zeros(1, np.uint32)
        assert lib.hfz_dbg_warp_fnv(src.ctypes.data, n, out.ctypes.data) == 0
        assert int(out[0]) == serial(en.tolist(), True), n
        assert int(out[1]) == serial(en.tolist(), False), n
