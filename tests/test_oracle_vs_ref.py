"""The plain-C restatement (oracle/hfz_oracle.c) against the compiled, unmodified reference
(oracle/_ref) on randomized inputs.  Skipped when the reference is not built."""
import numpy as np
import pytest

from oracle import pyoracle
from paper_2603_12485_b200 import synth

S = 65536


def test_feedback_random(port, ref):
    for raw, n in ((synth.maps_iid(96, S, seed=5), 96), (synth.maps_campaign(192, S, seed=6, p_extra=8, p_rare=8), 192),
                   synth.maps_edge_cases(S)):
        outs = []
        for ck in (port, ref):
            v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
            o = ck.feedback_batch(raw, n, S, v, c, want_classed=True)
            outs.append((o, v, c))
        (a, av, ac), (b, bv, bc) = outs
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(av, bv) and np.array_equal(ac, bc)


def test_feedback_262144(port):
    S2 = 262144
    if not pyoracle.Ref.available(S2):
        pytest.skip("262,144-slot reference build absent")
    r2 = pyoracle.Ref(S2)
    raw = synth.maps_iid(12, S2, density=0.01, seed=8)
    outs = []
    for ck in (port, r2):
        v, c = np.zeros(S2, np.uint8), np.zeros(2, np.uint64)
        outs.append((ck.feedback_batch(raw, 12, S2, v, c, want_classed=True), v, c))
    for k in outs[0][0]:
        assert np.array_equal(outs[0][0][k], outs[1][0][k]), k
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][2], outs[1][2])


def test_havoc_random(port, ref):
    rng = np.random.default_rng(1)
    for i in range(600):
        ln = int(rng.integers(0, 40)) if i % 3 else int(rng.integers(0, 3000))
        data = rng.integers(0, 256, ln, dtype=np.uint8).tobytes()
        seed = int(rng.integers(0, 2 ** 63))
        assert port.havoc(data, seed) == ref.havoc(data, seed), (i, ln, seed)
    for ln in (0, 1, 2, 3, 4, 5):
        for seed in range(40):
            data = bytes(range(ln))
            assert port.havoc(data, seed) == ref.havoc(data, seed)


def test_havoc_near_cap(port, ref):
    data = np.random.default_rng(2).integers(0, 256, (1 << 20) - 8, dtype=np.uint8).tobytes()
    for seed in (42, 43, 44):
        a, b = port.havoc(data, seed), ref.havoc(data, seed)
        assert a[1:] == b[1:] and a[0] == b[0]


def test_splice_deterministic_random(port, ref):
    rng = np.random.default_rng(3)
    for i in range(200):
        a = rng.integers(0, 256, int(rng.integers(0, 60)), dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, int(rng.integers(0, 60)), dtype=np.uint8).tobytes()
        seed = int(rng.integers(0, 2 ** 63))
        assert port.splice(a, b, seed) == ref.splice(a, b, seed)
    for ln in (0, 1, 2, 3, 4, 5, 8, 31, 32, 33, 70):
        d = rng.integers(0, 256, ln, dtype=np.uint8).tobytes()
        assert port.deterministic(d) == ref.deterministic(d)


def random_exec(rng, n_launch, three_d=False, max_len=12, n_sites=40):
    dims, ev_off, sites = [], [0], []
    for _ in range(n_launch):
        if three_d:
            g = (int(rng.integers(1, 3)), int(rng.integers(1, 4)), int(rng.integers(1, 3)))
            b = (int(rng.integers(1, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 4)))
        else:
            g = (int(rng.integers(1, 4)), 1, 1)
            b = (int(rng.integers(1, 100)), 1, 1)
        dims.append([*g, *b])
        threads = g[0] * g[1] * g[2] * b[0] * b[1] * b[2]
        pool = rng.integers(0, 2 ** 32, n_sites, dtype=np.uint64)
        shared = rng.integers(0, n_sites, int(rng.integers(1, max_len)))
        for t in range(threads):
            if rng.random() < 0.6:
                seq = shared
            else:
                seq = rng.integers(0, n_sites, int(rng.integers(0, max_len)))
            sites.extend(int(pool[i]) for i in seq)
            ev_off.append(len(sites))
    return np.array(dims, np.uint32), np.array(ev_off, np.uint64), np.array(sites, np.uint32)


def test_edge_record_random(port, ref):
    rng = np.random.default_rng(4)
    for i in range(60):
        d, e, s = random_exec(rng, int(rng.integers(1, 4)), three_d=bool(i % 2))
        a, ae = port.edge_record_exec(d, e, s)
        b, be = ref.edge_record_exec(d, e, s)
        assert np.array_equal(a, b) and ae == be, i


def test_edge_record_synth_batch(port, ref):
    tr = synth.bb_traces(2, grid=(2, 1, 1), block=(96, 1, 1), n_launch=3)
    raw, ev = port.edge_record_batch(tr["launch_off"], tr["dims"], tr["thread_off"], tr["ev_off"], tr["sites"], 2, S)
    rec = pyoracle.record_bytes(S)
    for e in range(2):
        l0, l1 = int(tr["launch_off"][e]), int(tr["launch_off"][e + 1])
        t0 = int(tr["thread_off"][l0])
        c, n = ref.edge_record_exec(tr["dims"][l0:l1], tr["ev_off"][t0:], tr["sites"])
        assert np.array_equal(raw[e * rec + S // 2:(e + 1) * rec].view(np.uint32), c) and n == ev[e]
