"""Seeded randomized differential test of the feedback fold: random batch sizes, densities from
empty to full, counts at ladder boundaries and extremes, random pre-warmed virgin maps, every
dense scan kernel and both sparse paths, all compared with the CPU oracle (classed bytes, Admit
codes in order, both signatures, nnz, final virgin, edge counters)."""
import numpy as np
import pytest
import torch

import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

pytestmark = pytest.mark.gpu

HOST_VALUES = np.array([1, 2, 3, 4, 7, 8, 15, 16, 31, 32, 127, 128, 255], np.uint8)
DEV_VALUES = np.array([1, 2, 3, 511, 512, 4095, 4096, 16383, 16384, 65535, 65536, 0x7FFFFFFF, 0xFFFFFFFF], np.uint32)
KERNELS = {"lane_per_map": (0, 0, 0, 0), "warp_per_map": (1 << 40, 0, 0, 0), "pipelined": (0, 1 << 20, 0, 0),
           "two_stage": (0, 0, 1 << 40, 0), "fused_step": (0, 0, 1 << 40, 1), "auto": (-1, -1, -1, 1)}


def random_batch(rng, n, S):
    """n raw records with per-map densities spread over several orders of magnitude."""
    H = S // 2
    raw = np.zeros(n * synth.record_bytes(S), np.uint8)
    rec = raw.reshape(n, -1)
    host, dev = rec[:, :H], rec[:, H:].view(np.uint32)
    shared = rng.integers(0, S, max(1, S // 200))            # slots many maps have in common
    for e in range(n):
        kind = rng.integers(0, 6)
        if kind == 0:
            continue                                          # empty map
        dens = [0.0005, 0.005, 0.02, 0.2, 1.0][kind - 1]
        k = max(1, int(dens * S))
        idx = rng.integers(0, S, k) if dens < 1.0 else np.arange(S)
        if rng.random() < 0.7:
            idx = np.concatenate([idx, shared[: rng.integers(1, len(shared) + 1)]])
        hi = idx[idx < H]
        di = idx[idx >= H] - H
        host[e, hi] = HOST_VALUES[rng.integers(0, len(HOST_VALUES), hi.size)]
        dev[e, di] = DEV_VALUES[rng.integers(0, len(DEV_VALUES), di.size)]
    return raw


@pytest.mark.parametrize("seed", range(24))
def test_random_batches_against_the_oracle(seed, port):
    rng = np.random.default_rng(1000 + seed)
    S = int(rng.choice([1024, 4096, 65536, 65536, 65536]))
    n = int(rng.choice([1, 2, 31, 33, 64, 100, 257]))
    raw = random_batch(rng, n, S)
    # a random pre-warmed virgin map, with consistent edge counters
    v0 = np.zeros(S, np.uint8)
    warm = rng.integers(0, S, int(rng.integers(0, S // 4)))
    v0[warm] = rng.integers(1, 256, warm.size).astype(np.uint8)
    c0 = np.array([np.count_nonzero(v0[: S // 2]), np.count_nonzero(v0[S // 2:])], np.uint64)
    wv, wc = v0.copy(), c0.copy()
    want = port.feedback_batch(raw, n, S, wv, wc, want_classed=True)

    ctx = hfz.Context(0, S)
    try:
        kname = list(KERNELS)[seed % len(KERNELS)]
        for key, val in zip(("scan_small", "scan_pipe", "scan_two_stage", "small_fused"), KERNELS[kname]):
            ctx.set_option(key, val)
        ctx.set_option("sparse_native", seed % 2)
        # dense, device buffers
        virgin = torch.from_numpy(v0).to(ctx.device)
        counts = torch.from_numpy(c0.view(np.int64)).to(ctx.device)
        o = ctx.feedback_batch(torch.from_numpy(raw).to(ctx.device), virgin, counts, want_classed=True)
        ctx.synchronize()
        got = dict(admit=o["admit"].cpu().numpy(), sig_full=o["sig_full"].cpu().numpy().view(np.uint64),
                   sig_simple=o["sig_simple"].cpu().numpy().view(np.uint64),
                   nnz=o["nnz"].cpu().numpy().view(np.uint32), classed=o["classed"].cpu().numpy())
        for k in want:
            assert np.array_equal(got[k], want[k]), f"dense/{kname}: {k} differs (S={S}, n={n})"
        assert np.array_equal(virgin.cpu().numpy(), wv) and np.array_equal(counts.cpu().numpy().view(np.uint64), wc)
        # sparse, host buffers (pairs in random order)
        entries, off = synth.to_sparse(raw, n, S, shuffle_seed=seed)
        v, c = v0.copy(), c0.copy()
        sp = ctx.feedback_batch_sparse_host(entries, off, v, c, want_classed=True)
        for k in want:
            assert np.array_equal(sp[k], want[k]), f"sparse/native={seed % 2}: {k} differs (S={S}, n={n})"
        assert np.array_equal(v, wv) and np.array_equal(c, wc)
    finally:
        ctx.close()
