#!/usr/bin/env python
"""Randomized soak of every kernel family against the CPU oracle (many more seeds than the test
suite runs): the fold (all scan kernels, dense + sparse + compact), edge record (uniform and
mixed launch geometries, divergent warps, loops), havoc / splice.  Prints one line per family;
exits non-zero on the first mismatch.

    python scripts/soak.py [--seeds N]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2603_12485_b200 as hfz
from oracle import pyoracle
from paper_2603_12485_b200 import synth
from tests import test_fuzz_gpu as fz
from tests.test_edge_record_gpu import pack
from tests.test_mutators_gpu import check_havoc
from tests.test_oracle_vs_ref import random_exec


def soak_fold(seeds, port):
    t = time.time()
    for seed in range(100, 100 + seeds):
        fz.test_random_batches_against_the_oracle.__wrapped__(seed, port) if hasattr(
            fz.test_random_batches_against_the_oracle, "__wrapped__") else fz.test_random_batches_against_the_oracle(seed, port)
    # compact lists on the same kind of batches
    for seed in range(seeds // 4):
        rng = np.random.default_rng(5000 + seed)
        n = int(rng.choice([1, 33, 100]))
        raw = fz.random_batch(rng, n, 65536)
        comp, coff, wide, woff = synth.to_compact(raw, n, 65536, shuffle_seed=seed)
        v, c = np.zeros(65536, np.uint8), np.zeros(2, np.uint64)
        ctx = hfz.Context(0)
        got = ctx.feedback_batch_compact_host(comp, coff, wide if wide.shape[0] else None,
                                              woff if wide.shape[0] else None, v, c, want_classed=True)
        # and the packed form of the same batch (3-byte host entries, 17-bit device counts)
        h3, hoff, d17, doff = synth.to_packed(raw, n, 65536, shuffle_seed=seed + 1)
        v2, c2 = np.zeros(65536, np.uint8), np.zeros(2, np.uint64)
        got2 = ctx.feedback_batch_packed_host(h3, hoff, d17, doff, v2, c2, want_classed=True)
        ctx.close()
        wv, wc = np.zeros(65536, np.uint8), np.zeros(2, np.uint64)
        want = port.feedback_batch(raw, n, 65536, wv, wc, want_classed=True)
        for k in want:
            assert np.array_equal(got[k], want[k]), (seed, k)
            assert np.array_equal(got2[k], want[k]), (seed, k, "packed")
        assert np.array_equal(v, wv) and np.array_equal(c, wc)
        assert np.array_equal(v2, wv) and np.array_equal(c2, wc)
    print(f"fold: {seeds} random batches x (dense + sparse) + {seeds // 4} compact and packed ok in {time.time() - t:.0f} s", flush=True)


def soak_edge(seeds, port):
    t = time.time()
    ctx = hfz.Context(0)
    S = 65536
    for seed in range(seeds):
        rng = np.random.default_rng(9000 + seed)
        execs = []
        for i in range(24):
            style = rng.integers(0, 4)
            if style == 0:      # mixed geometries
                execs.append(random_exec(rng, int(rng.integers(1, 5)), three_d=bool(i % 2), max_len=int(rng.integers(2, 40)),
                                         n_sites=int(rng.integers(2, 600))))
            else:               # uniform geometry over several launches, idle threads, loops, divergence
                d = [int(rng.integers(1, 4)), int(rng.integers(1, 3)), 1, int(rng.integers(1, 130)), 1, 1]
                threads = d[0] * d[1] * d[3]
                nl = int(rng.integers(1, 5))
                pool = rng.integers(0, 2 ** 32, int(rng.integers(1, 700)), dtype=np.uint64)
                if rng.random() < 0.3:
                    pool[0] = 0xFFFFFFFF
                common = pool[rng.integers(0, len(pool), int(rng.integers(1, 20)))]
                ev, sites = [0], []
                for _ in range(nl):
                    for _t in range(threads):
                        r = rng.random()
                        if r < 0.2:
                            seq = []
                        elif r < 0.7:
                            seq = common
                        elif r < 0.85:
                            seq = np.repeat(pool[rng.integers(0, len(pool), 2)], int(rng.integers(1, 40)))  # loops
                        else:
                            seq = pool[rng.integers(0, len(pool), int(rng.integers(1, 30)))]
                        sites.extend(int(x) for x in seq)
                        ev.append(len(sites))
                execs.append((np.array([d] * nl, np.uint32), ev, sites))
        tr = pack(execs)
        i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(ctx.device)
        sites = np.ascontiguousarray(tr["sites"], np.uint32)
        if sites.size == 0:
            sites = np.zeros(1, np.uint32)
        raw, ev = ctx.edge_record_batch(i64(tr["launch_off"]),
                                        torch.from_numpy(np.ascontiguousarray(tr["dims"], np.uint32).view(np.int32)).to(ctx.device),
                                        i64(tr["thread_off"]), i64(tr["ev_off"]),
                                        torch.from_numpy(sites.view(np.int32)).to(ctx.device), len(execs))
        ctx.synchronize()
        want_raw, want_ev = port.edge_record_batch(tr["launch_off"], tr["dims"], tr["thread_off"], tr["ev_off"],
                                                   tr["sites"], len(execs), S)
        assert np.array_equal(ev.cpu().numpy().view(np.uint64), want_ev), seed
        assert np.array_equal(raw.cpu().numpy(), want_raw), seed
        # the list output of the same batch: every listed exec's pairs are its device half, the others
        # (launches of differing geometry, too many distinct slots) are reported as not listed
        cap = int(rng.choice([64, 700, 4096]))
        o = ctx.edge_record_batch_lists(i64(tr["launch_off"]),
                                        torch.from_numpy(np.ascontiguousarray(tr["dims"], np.uint32).view(np.int32)).to(ctx.device),
                                        i64(tr["thread_off"]), i64(tr["ev_off"]),
                                        torch.from_numpy(sites.view(np.int32)).to(ctx.device), len(execs), cap=cap)
        ctx.synchronize()
        ent = o["entries"].cpu().numpy().view(np.uint32).reshape(len(execs), cap, 2)
        ns = o["n_slots"].cpu().numpy()
        dev = want_raw.reshape(len(execs), synth.record_bytes(S))[:, S // 2:].view(np.uint32)
        listed = 0
        for e in range(len(execs)):
            nz = np.nonzero(dev[e])[0]
            if ns[e] < 0:
                assert not ent[e].any(), (seed, e)
                continue
            listed += 1
            assert ns[e] == nz.size and nz.size <= cap, (seed, e)
            got = {int(a): int(b) for a, b in ent[e, :ns[e]]}
            assert got == {int(S // 2 + k): int(dev[e][k]) for k in nz} and not ent[e, ns[e]:].any(), (seed, e)
        n_listed_total = listed if seed == 0 else n_listed_total + listed
    ctx.close()
    print(f"edge record lists: {n_listed_total} of {seeds * 24} execs listed, all equal to their dense halves", flush=True)
    print(f"edge record: {seeds} random batches of 24 execs ok in {time.time() - t:.0f} s", flush=True)


def soak_havoc(seeds, checker):
    t = time.time()
    ctx = hfz.Context(0)
    for seed in range(seeds):
        rng = np.random.default_rng(20000 + seed)
        inputs = [rng.integers(0, 256, int(rng.choice([0, 1, 2, 3, 4, 5, 17, 64, 300, 2000, 5000, 7000])), dtype=np.uint8).tobytes()
                  for _ in range(48)]
        states = [int(x) for x in rng.integers(0, 2 ** 63, 48, dtype=np.uint64)]
        check_havoc(ctx, checker, inputs, states)
    ctx.close()
    print(f"havoc: {seeds} random batches of 48 inputs ok in {time.time() - t:.0f} s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    a = ap.parse_args()
    port = pyoracle.Port()
    checker = pyoracle.best_checker()
    soak_fold(a.seeds, port)
    soak_edge(max(1, a.seeds // 2), port)
    soak_havoc(max(1, a.seeds // 2), checker)
    print("soak: all families ok")
