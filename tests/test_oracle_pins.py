"""The CPU oracles pinned against the reference's own known-answer tests.

Every case restates a test of /root/reference/proj/tests and runs against BOTH checkers: the
plain-C restatement (oracle/hfz_oracle.c) and, when it was built, the compiled reference
(oracle/_ref).  Values in hex were produced by the compiled reference during the survey.
"""
import numpy as np
import pytest

from oracle import pyoracle

S, H = 65536, 32768
REC = pyoracle.record_bytes(S)


def checkers():
    out = [pytest.param("port", id="port")]
    out.append(pytest.param("ref", id="ref"))
    return out


@pytest.fixture(params=["port", "ref"])
def ck(request):
    if request.param == "port":
        return pyoracle.Port()
    if not pyoracle.Ref.available():
        pytest.skip("oracle/_ref not built")
    return pyoracle.Ref()


def mk(host=(), dev=()):
    r = np.zeros(REC, np.uint8)
    for i, v in host:
        r[i] = v
    d = r[H:].view(np.uint32)
    for i, v in dev:
        d[i - H] = v
    return r


def fold(ck, maps, virgin=None, counts=None):
    raw = np.concatenate(maps)
    v = np.zeros(S, np.uint8) if virgin is None else virgin
    c = np.zeros(2, np.uint64) if counts is None else counts
    o = ck.feedback_batch(raw, len(maps), S, v, c, want_classed=True)
    return o, v, c


def host_class(c):
    if c == 0: return 0
    if c == 1: return 1
    if c == 2: return 2
    if c == 3: return 4
    if c <= 7: return 8
    if c <= 15: return 16
    if c <= 31: return 32
    if c <= 127: return 64
    return 128


def dev_class(c):
    if c == 0: return 0
    if c == 1: return 1
    if c == 2: return 2
    if c <= 511: return 4
    if c <= 4095: return 8
    if c <= 16383: return 16
    if c <= 65535: return 32
    return 64


def test_ladders_exhaustive(ck):
    """tests/test_coverage.cpp:119-130 and tests/acceptance.cpp:303-321 (0..200,000 + extremes)."""
    step = 1 if ck.kind == "port" else 7  # the ctypes round trip is the cost; port is checked exhaustively
    for c in list(range(0, 200001, step)) + [0x7FFFFFFF, 0xFFFFFFFF, (1 << 64) - 1]:
        assert ck.classify_host(c) == host_class(c), c
        assert ck.classify_device(c) == dev_class(c), c
    for c in [1, 2, 3, 4, 7, 8, 15, 16, 31, 32, 127, 128, 511, 512, 4095, 4096, 16383, 16384, 65535, 65536]:
        assert ck.classify_host(c) == host_class(c) and ck.classify_device(c) == dev_class(c)


def test_device_edge_index(ck):
    """tests/test_coverage.cpp:145-155: 10,000 random pairs from Rng(0x77)."""
    st = 0x77
    for _ in range(10000):
        a, st = ck.rng_next(st)
        b, st = ck.rng_next(st)
        a &= 0xFFFFFFFF
        b &= 0xFFFFFFFF
        idx = ck.device_edge_index(a, b)
        assert H <= idx < S and idx == H + ((a ^ b) % 32768)


def test_classify_example(ck):
    """tests/test_coverage.cpp:157-175."""
    o, _, _ = fold(ck, [mk(host=[(10, 1), (500, 5)], dev=[(H + 3, 700), (S - 1, 2)])])
    assert np.nonzero(o["classed"][0])[0].tolist() == [10, 500, H + 3, S - 1]
    assert o["classed"][0][[10, 500, H + 3, S - 1]].tolist() == [1, 8, 8, 2]
    assert o["nnz"][0] == 4


def test_admit_sequence(ck):
    """tests/test_coverage.cpp:177-221: NewEdges / None / NewCounts, new edge beats new count."""
    seq = [mk(host=[(42, 1)]), mk(host=[(42, 1)]), mk(host=[(42, 2)]), mk(host=[(42, 4)]),
           mk(host=[(42, 5)]), mk(host=[(42, 3), (43, 1)]), mk(dev=[(H + 9, 1)])]
    o, v, c = fold(ck, seq)
    assert o["admit"].tolist() == [2, 0, 1, 1, 0, 2, 2]
    assert c.tolist() == [2, 1]


def test_or_folding(ck):
    """tests/test_coverage.cpp:223-237."""
    o, v, c = fold(ck, [mk(host=[(100, 9)], dev=[(H + 5, 600)]), mk(host=[(100, 1)])])
    assert v[100] == (host_class(9) | host_class(1)) and v[H + 5] == dev_class(600)


def test_signatures(ck):
    """tests/test_coverage.cpp:239-259: byte-level FNV-1a, empty map = offset basis."""
    def fnv(bs):
        h = 14695981039346656037
        for b in bs:
            h = ((h ^ b) * 1099511628211) & ((1 << 64) - 1)
        return h
    o, _, _ = fold(ck, [mk(host=[(5, 3)], dev=[(40000, 700)]), mk()])
    assert int(o["sig_simple"][0]) == fnv([5, 0, 40000 & 0xFF, 40000 >> 8]) == 0x2E1A3655EF7B3874
    assert int(o["sig_full"][0]) == fnv([5, 0, 4, 40000 & 0xFF, 40000 >> 8, 8]) == 0x31CF681E15834C40
    assert int(o["sig_simple"][1]) == int(o["sig_full"][1]) == 0xCBF29CE484222325


def test_full_refines_simple(ck):
    """tests/test_coverage.cpp:261-289."""
    o, _, _ = fold(ck, [mk(host=[(9, 1)]), mk(host=[(9, 2)])])
    assert o["sig_simple"][0] == o["sig_simple"][1] and o["sig_full"][0] != o["sig_full"][1]
    st = 0xABC
    f2s = {}
    maps = []
    for _ in range(300):
        m = {}
        e, st = ck.rng_below(st, 6)
        for _ in range(1 + e):
            slot, st = ck.rng_below(st, 64)
            hits, st = ck.rng_below(st, 5)
            m[slot] = m.get(slot, 0) + 1 + hits
        maps.append(mk(host=list(m.items())))
    o, _, _ = fold(ck, maps)
    for fs, ss in zip(o["sig_full"].tolist(), o["sig_simple"].tolist()):
        assert f2s.setdefault(fs, ss) == ss


def test_splitmix64_known_answers(ck):
    """outputs of the compiled reference."""
    st = 0
    outs = []
    for _ in range(3):
        v, st = ck.rng_next(st)
        outs.append(v)
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    st = 1
    outs = []
    for _ in range(3):
        v, st = ck.rng_next(st)
        outs.append(v)
    assert outs == [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E]
    # below(n<=1) draws nothing (rng.hpp:25); jump-ahead: state after k draws = seed + k*gamma
    v, st2 = ck.rng_below(5, 1)
    assert v == 0 and st2 == 5
    st = 99
    for k in range(1, 50):
        _, st = ck.rng_next(st)
        assert st == (99 + k * pyoracle.GAMMA) & pyoracle.MASK64


def test_rng_bounds_and_split(ck):
    """tests/test_coverage.cpp:311-332."""
    st = 7
    for _ in range(2000):
        n, st = ck.rng_below(st, 1000)
        v, st = ck.rng_below(st, n + 1)
        assert v < n + 1
    c1, st = ck.rng_split(123, 1)
    c2, st = ck.rng_split(st, 2)
    assert c1 != c2


def test_havoc_known_answers(ck):
    """byte strings produced by the compiled reference."""
    if ck.kind == "reference" and not ck.has_engine:
        pytest.skip("engine not in this build")
    base = bytes(range(16))
    out, st, draws = ck.havoc(base, 1)
    assert out.hex() == "bcffbcbc000301" and draws == 117
    out, st, draws = ck.havoc(base, 2)
    assert out.hex() == "a10080220080000102d9d9e57f0202ff7f02f78bff15d90c0000800000d90287" and draws == 126
    out, st, draws = ck.havoc(b"", 1)
    assert out.hex() == "ff00027f19" and draws == 120
    out, st, draws = ck.havoc(bytes(8), 7)
    assert out.hex() == "0002ff05f4" and draws == 73
    # tests/test_engine.cpp:128-152: reproducible per seed, seeds differ, grows empty input, 1 MiB cap
    assert ck.havoc(base, 7)[0] == ck.havoc(base, 7)[0]
    assert ck.havoc(bytes(64), 7)[0] != ck.havoc(bytes(64), 8)[0]
    assert len(ck.havoc(b"", 3)[0]) >= 1
    big = bytes(1 << 20)
    assert len(ck.havoc(big, 42)[0]) <= 1 << 20


def test_splice_and_deterministic(ck):
    """tests/test_engine.cpp:85-126,154-169; python smoke test_smoke.py:53-60."""
    if ck.kind == "reference" and not ck.has_engine:
        pytest.skip("engine not in this build")
    assert ck.splice(b"AAAAAAAA", b"BBBBBBBB", 7)[0] == b"AAABBBBBBBB"
    ms = ck.deterministic(bytes(8))
    assert len(ms) == 1638 and ms[0] == b"\x80" + bytes(7) and len(set(ms)) > 500
    first = [m[0] for m in ms[:8]]
    assert first == [0x80, 0x40, 0x20, 0x10, 0x08, 0x04, 0x02, 0x01]
    assert ms[64][0] == 1 and ms[65][0] == 0xFF and ms[66][0] == 2 and ms[67][0] == 0xFE  # +1,-1,+2,-2
    assert ck.deterministic(b"") == []
    # window: offsets capped to the first 32 bytes
    ms = ck.deterministic(bytes(100))
    assert all(m[40:] == bytes(60) for m in ms)


def test_host_edge_chain(ck):
    """tests/test_coverage.cpp:77-117: chain vs sparse replay, never-zero pinning."""
    st = 0x1234
    for _ in range(20):
        ln, st = ck.rng_below(st, 400)
        sites = []
        for _ in range(1 + ln):
            s, st = ck.rng_below(st, H)
            sites.append(s)
        half, viol = ck.host_edge_record(np.array(sites, np.uint16))
        counts = {}
        prev = 0
        for s in sites:
            counts[prev ^ s] = counts.get(prev ^ s, 0) + 1
            prev = s >> 1
        want = np.zeros(H, np.uint8)
        for k, n in counts.items():
            want[k] = (n - 1) % 255 + 1
        assert np.array_equal(half, want) and viol == 0
    half, _ = ck.host_edge_record(np.zeros(1000, np.uint16))  # site 0 forever: slot 0, 1000 hits
    assert half[0] == (1000 - 1) % 255 + 1 and half[1:].sum() == 0


def chain_exec(ck, block, launches, grid=(1, 1, 1)):
    tpb = block[0] * block[1] * block[2]
    threads = tpb * grid[0] * grid[1] * grid[2]
    dims, ev_off, sites = [], [0], []
    for ch in launches:
        dims.append([*grid, *block])
        for _ in range(threads):
            sites.extend(ch)
            ev_off.append(len(sites))
    return ck.edge_record_exec(np.array(dims, np.uint32), np.array(ev_off, np.uint64),
                               np.array(sites, np.uint32))


def chain_oracle(blocks, tpb, launches):
    warps = blocks * ((tpb + 31) // 32)
    counts = {}
    prev = 0
    for ch in launches:
        for s in ch:
            slot = (prev ^ s) % 32768
            counts[slot] = counts.get(slot, 0) + warps
            prev = s >> 1
    return counts


def check_counts(counters, want):
    got = {int(i): int(counters[i]) for i in np.nonzero(counters)[0]}
    assert got == want


def test_warp_counting(ck):
    """tests/test_hdvm.cpp:89-127 and acceptance criterion 5 (tests/acceptance.cpp:266-299)."""
    for t in (1, 31, 32, 33, 64, 100, 1024):
        c, ev = chain_exec(ck, (t, 1, 1), [[11, 29, 11, 500]])
        check_counts(c, chain_oracle(1, t, [[11, 29, 11, 500]]))
        assert ev == 4 * ((t + 31) // 32)
    c, _ = chain_exec(ck, (33, 1, 1), [[7]])
    assert c[7] == 2
    c, _ = chain_exec(ck, (40, 1, 1), [[3, 9]], grid=(2, 2, 1))
    check_counts(c, chain_oracle(4, 40, [[3, 9]]))
    launches = [[5, 6], [6, 5, 6]]  # prev carries across launches
    c, _ = chain_exec(ck, (8, 1, 1), launches)
    check_counts(c, chain_oracle(1, 8, launches))
    for t in (1, 31, 32, 33, 64, 100, 1024):
        c, _ = chain_exec(ck, (t, 1, 1), [[7777]])
        assert c[7777 % 32768] == (t + 31) // 32


def test_divergent_and_loop(ck):
    """tests/test_hdvm.cpp:129-187: a single divergent thread, forked lanes, the loop case."""
    # thread 5 of 32 takes an extra site: exactly one bump for it
    dims = np.array([[1, 1, 1, 32, 1, 1]], np.uint32)
    sites, ev = [], [0]
    for t in range(32):
        sites += [10, 999] if t == 5 else [10]
        ev.append(len(sites))
    c, n = ck.edge_record_exec(dims, np.array(ev, np.uint64), np.array(sites, np.uint32))
    assert n == 2 and c[10] == 1 and c[((10 >> 1) ^ 999) % 32768] == 1
    # loop: lane L visits site 77 (L % 31) + 1 times -> 31 bumps, slot(77) once, slot((77>>1)^77) 30 times
    sites, ev = [], [0]
    for t in range(32):
        sites += [77] * ((t % 31) + 1)
        ev.append(len(sites))
    c, n = ck.edge_record_exec(dims, np.array(ev, np.uint64), np.array(sites, np.uint32))
    assert n == 31 and c[77] == 1 and c[(77 >> 1) ^ 77] == 30
