#!/usr/bin/env python
"""Probe of the sparse ingest path: host-buffer call and device-buffer call at several chunk sizes
(bench.py's workload, 65,536 execs unless --execs)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
import paper_2603_12485_b200 as hfz


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--execs", type=int, default=65536)
    ap.add_argument("--chunks", default="2048,4096,8192,16384")
    args = ap.parse_args()
    n, S, REC = args.execs, bench.S, bench.REC
    dev = torch.device("cuda", 0)
    raw = torch.empty(n * REC, dtype=torch.uint8, device=dev)
    for i in range(0, n, 4096):
        m = min(4096, n - i)
        raw[i * REC:(i + m) * REC] = torch.from_numpy(bench.make_maps(m, i, "campaign")).to(dev)
    ctx0 = hfz.Context(0, S)
    virgin, counts = ctx0.new_virgin(), ctx0.new_edge_counts()
    ctx0.feedback_batch(torch.from_numpy(bench.make_maps(4096, 1 << 24, "campaign")).to(dev), virgin, counts)
    v0, c0 = virgin.cpu().numpy(), counts.cpu().numpy().view(np.uint64)
    ent_t, off_t = bench.sparse_lists_from_device(raw, n, dev)
    ent_np, off_np = ent_t.numpy().view(np.uint32), off_t.numpy().view(np.uint64)
    ent_d, off_d = ent_t.to(dev), off_t.to(dev)
    comp_t, coff_t, wide_t, woff_t = bench.compact_lists(ent_t, off_t)
    comp_np, coff_np = comp_t.numpy().view(np.uint32), coff_t.numpy().view(np.uint64)
    wide_np, woff_np = wide_t.numpy().view(np.uint32), woff_t.numpy().view(np.uint64)
    print(f"{n} execs, {ent_np.shape[0] / n:.1f} pairs/exec, {ent_np.nbytes / 1e6:.1f} MB of pairs")
    ctx0.close()
    for chunk in [int(x) for x in args.chunks.split(",")]:
        ctx = hfz.Context(0, S)
        ctx.set_option("sparse_chunk", chunk)
        ts = []
        for i in range(4):
            vh, ch = v0.copy(), c0.copy()
            torch.cuda.synchronize()
            t = time.perf_counter()
            ctx.feedback_batch_sparse_host(ent_np, off_np, vh, ch)
            ts.append(time.perf_counter() - t)
        host_ms = min(ts[1:]) * 1e3
        ts = []
        for i in range(4):
            vh, ch = v0.copy(), c0.copy()
            torch.cuda.synchronize()
            t = time.perf_counter()
            ctx.feedback_batch_compact_host(comp_np, coff_np, wide_np, woff_np, vh, ch)
            ts.append(time.perf_counter() - t)
        comp_ms = min(ts[1:]) * 1e3
        vd, cd = torch.from_numpy(v0).to(dev), torch.from_numpy(c0.view(np.int64)).to(dev)
        out = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(3):
            vd.copy_(torch.from_numpy(v0))
            torch.cuda.synchronize()
            e0.record()
            out = ctx.feedback_batch_sparse(ent_d, off_d, vd, cd, out=out)
            e1.record()
            torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1)
        print(f"chunk {chunk:6d}: host call {host_ms:7.2f} ms ({n / host_ms / 1e3:.2f} M evals/s, "
              f"{ent_np.nbytes / host_ms / 1e6:.1f} GB/s of pairs) | compact host call {comp_ms:6.2f} ms "
              f"({n / comp_ms / 1e3:.2f} M evals/s) | device call {dev_ms:6.2f} ms "
              f"({n / dev_ms / 1e3:.2f} M evals/s)")
        ctx.close()


if __name__ == "__main__":
    main()
