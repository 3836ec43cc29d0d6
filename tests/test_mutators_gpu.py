"""K3 parity: batched havoc / splice / deterministic on the GPU vs the CPU oracle, byte for byte,
including end Rng states and draw counts."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import api, synth

pytestmark = pytest.mark.gpu
GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def gpu_havoc(ctx, inputs, states):
    n = len(inputs)
    lens = np.array([len(b) for b in inputs], np.int64)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    blob = np.frombuffer(b"".join(inputs) + bytes(16), np.uint8).copy()
    d_state = torch.from_numpy(api.u64_to_i64(np.array(states, np.uint64))).to(ctx.device)
    ob, oo, ol, dr = ctx.havoc_batch(torch.from_numpy(blob).to(ctx.device), torch.from_numpy(off).to(ctx.device), d_state)
    ctx.synchronize()
    ob, oo, ol = ob.cpu().numpy(), oo.cpu().numpy(), ol.cpu().numpy()
    outs = [ob[oo[j]:oo[j] + ol[j]].tobytes() for j in range(n)]
    return outs, api.i64_to_u64(d_state).tolist(), dr.cpu().numpy().tolist()


def check_havoc(ctx, checker, inputs, states):
    outs, ends, draws = gpu_havoc(ctx, inputs, states)
    for j, (data, st) in enumerate(zip(inputs, states)):
        want, wst, wdr = checker.havoc(data, st)
        assert outs[j] == want, f"slot {j} len {len(data)} state {st:#x}"
        assert ends[j] == wst and draws[j] == wdr, f"slot {j}: state/draws"


def test_known_answers(ctx):
    """SURVEY 8c byte strings (compiled reference) through the reference-named Python API."""
    assert hfz.havoc_mutant(bytes(range(16)), 1).hex() == "bcffbcbc000301"
    assert hfz.havoc_mutant(bytes(range(16)), 2).hex() == "a10080220080000102d9d9e57f0202ff7f02f78bff15d90c0000800000d90287"
    assert hfz.havoc_mutant(b"", 1).hex() == "ff00027f19"
    assert hfz.havoc_mutant(bytes(8), 7).hex() == "0002ff05f4"
    assert hfz.splice_mutant(b"AAAAAAAA", b"BBBBBBBB", 7) == b"AAABBBBBBBB"
    ms = hfz.deterministic_mutants(bytes(8))
    assert len(ms) == 1638 and ms[0] == b"\x80" + bytes(7)
    assert hfz.deterministic_mutants(b"") == []
    assert hfz.MAP_SIZE == 65536 and hfz.HOST_SLOTS == 32768


def test_config4_fresh_seeds(ctx, checker):
    """1-4 KB inputs, slot j uses a fresh Rng(1000 + j) (the Python-API semantics)."""
    data, off = synth.havoc_inputs(1024, seed=45)
    inputs = [data[int(off[j]):int(off[j + 1])].tobytes() for j in range(1024)]
    check_havoc(ctx, checker, inputs, [1000 + j for j in range(1024)])


def test_config4_split_streams(ctx, checker):
    """Jump-ahead semantics: slot j uses parent.split(j) with parent = Rng(46); the parent state
    before slot j is 46 + j*gamma, so every child seed is an O(1) host computation."""
    data, off = synth.havoc_inputs(256, seed=47)
    inputs = [data[int(off[j]):int(off[j + 1])].tobytes() for j in range(256)]
    states = []
    for j in range(256):
        child, after = hfz.rng_split(hfz.rng_jump(46, j), j)
        assert after == hfz.rng_jump(46, j + 1)
        states.append(child)
    ref_parent = 46
    for j in range(4):  # the O(1) seeds equal the serial split chain of the oracle
        child, ref_parent = checker.rng_split(ref_parent, j)
        assert child == states[j]
    check_havoc(ctx, checker, inputs, states)


def test_edge_lengths(ctx, checker):
    rng = np.random.default_rng(5)
    inputs, states = [], []
    for ln in [0, 1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 33, 63, 64, 100, 255, 256, 1000, 5000, 5120, 5121, 9000]:
        for s in range(12):
            inputs.append(rng.integers(0, 256, ln, dtype=np.uint8).tobytes())
            states.append(int(rng.integers(0, 2 ** 63)) + s)
    check_havoc(ctx, checker, inputs, states)


def test_one_mib_inputs(ctx, checker):
    """kMaxInputBytes clamp (tests/test_engine.cpp:147-152): inputs at and just below 1 MiB work
    in the global-memory working buffer."""
    rng = np.random.default_rng(6)
    inputs = [rng.integers(0, 256, (1 << 20) - 8, dtype=np.uint8).tobytes(), bytes(1 << 20),
              rng.integers(0, 256, (1 << 20) - 1, dtype=np.uint8).tobytes()]
    outs, ends, draws = gpu_havoc(ctx, inputs, [42, 42, 7])
    for j, st in enumerate([42, 42, 7]):
        want, wst, wdr = checker.havoc(inputs[j], st)
        assert len(outs[j]) <= 1 << 20
        assert outs[j] == want and ends[j] == wst and draws[j] == wdr


def test_splice_batch(ctx, checker):
    rng = np.random.default_rng(7)
    inputs = [rng.integers(0, 256, int(rng.integers(0, 300)), dtype=np.uint8).tobytes() for _ in range(64)]
    inputs[3] = b""
    n = 200
    a_idx = rng.integers(0, 64, n).astype(np.int32)
    b_idx = rng.integers(0, 64, n).astype(np.int32)
    states = rng.integers(0, 2 ** 63, n).astype(np.uint64)
    lens = np.array([len(b) for b in inputs], np.int64)
    off = np.zeros(65, np.int64)
    np.cumsum(lens, out=off[1:])
    blob = np.frombuffer(b"".join(inputs) + bytes(16), np.uint8).copy()
    d_state = torch.from_numpy(api.u64_to_i64(states)).to(ctx.device)
    ob, oo, ol = ctx.splice_batch(torch.from_numpy(blob).to(ctx.device), torch.from_numpy(off).to(ctx.device),
                                  torch.from_numpy(a_idx).to(ctx.device), torch.from_numpy(b_idx).to(ctx.device), d_state)
    ctx.synchronize()
    ob, oo, ol = ob.cpu().numpy(), oo.cpu().numpy(), ol.cpu().numpy()
    ends = api.i64_to_u64(d_state)
    for j in range(n):
        want, wst = checker.splice(inputs[a_idx[j]], inputs[b_idx[j]], int(states[j]))
        assert ob[oo[j]:oo[j] + ol[j]].tobytes() == want and int(ends[j]) == wst


@pytest.mark.parametrize("ln", [1, 2, 3, 4, 5, 8, 31, 32, 33, 100])
def test_deterministic(ctx, checker, ln):
    data = np.random.default_rng(ln).integers(0, 256, ln, dtype=np.uint8).tobytes()
    assert hfz.deterministic_mutants(data) == checker.deterministic(data)
