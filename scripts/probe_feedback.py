"""Dev probe: time the fused feedback step for scan variants / warp counts (not a bench line)."""
import argparse
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--ns", default="", help="comma separated batch sizes to time with the defaults (prefixes of the generated batch)")
ap.add_argument("--mode", default="campaign")
ap.add_argument("--configs", default="row=512;row=256", help="; separated, each k=v,k=v over scan_row/scan_warps/scan_prefetch/virgin_smem")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sweep", default="", help="comma separated batch sizes: time every scan kernel on each")
a = ap.parse_args()
S = 65536
ctx = hfz.Context(0, S)
rec = ctx.rec
t = time.time()
chunk = 2048
raw = torch.empty(a.n * rec, dtype=torch.uint8, device=ctx.device)
gen = synth.maps_campaign if a.mode == "campaign" else synth.maps_iid
for i in range(0, a.n, chunk):
    m = min(chunk, a.n - i)
    raw[i * rec:(i + m) * rec] = torch.from_numpy(gen(m, S, first=i)).to(ctx.device)
print(f"generated {a.n} maps in {time.time()-t:.1f}s", flush=True)
virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
warm = torch.from_numpy(gen(4096, S, first=1 << 20)).to(ctx.device)
ctx.feedback_batch(warm, virgin, counts)
v0 = virgin.clone()
ALIAS = dict(row="scan_row", warps="scan_warps", prefetch="scan_prefetch", vsmem="virgin_smem")
DEFAULTS = dict(scan_row=0, scan_warps=0, scan_prefetch=1, virgin_smem=1)
for cfg in a.configs.split(";"):
    opts = dict(DEFAULTS)
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        opts[ALIAS.get(k, k)] = int(v)
    for k, v in opts.items():
        ctx.set_option(k, v)
    out = None
    ts = []
    for r in range(a.reps + 2):
        virgin.copy_(v0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = ctx.feedback_batch(raw, virgin, counts, out=out)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    cand = int((out["admit"] != 0).sum())
    print(f"{cfg:40s}: {ms:8.3f} ms  {a.n/ms*1e3/1e6:7.3f} M evals/s  "
          f"{a.n*rec/ms/1e6:8.1f} GB/s ({a.n*rec/ms/1e6/6544.7*100:4.1f}% of 6544.7)  admits {cand}", flush=True)

if a.ns:
    for k, v in DEFAULTS.items():
        ctx.set_option(k, v)
    for n in [int(x) for x in a.ns.split(",")]:
        sub = raw[: n * rec]
        ts = []
        for r in range(a.reps + 2):
            virgin.copy_(v0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            o = ctx.feedback_batch(sub, virgin, counts)
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        print(f"n={n:7d}: {ms:8.3f} ms  {n/ms*1e3/1e6:7.3f} M evals/s  {n*rec/ms/1e6:8.1f} GB/s ({n*rec/ms/1e6/6544.7*100:4.1f}%)", flush=True)

if a.sweep:
    KERN = {"lane": dict(scan_small=0, scan_pipe=0, scan_two_stage=0), "wpm": dict(scan_small=1 << 40, scan_pipe=0, scan_two_stage=0),
            "pipe512": dict(scan_small=0, scan_pipe=1 << 20, scan_row=512, scan_two_stage=0),
            "pipe256": dict(scan_small=0, scan_pipe=1 << 20, scan_row=256, scan_two_stage=0),
            "two": dict(scan_small=0, scan_pipe=0, scan_two_stage=1 << 40),
            "auto": dict(scan_small=-1, scan_pipe=-1, scan_two_stage=-1)}
    for n in [int(x) for x in a.sweep.split(",")]:
        sub = raw[: n * rec]
        line = f"n={n:7d} ideal {n*rec/6544.7e6:6.3f} ms |"
        for name, opts in KERN.items():
            for k, v in dict(DEFAULTS, **opts).items():
                ctx.set_option(k, v)
            ts = []
            for r in range(a.reps + 2):
                virgin.copy_(v0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                o = ctx.feedback_batch(sub, virgin, counts)
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            line += f" {name} {min(ts):6.3f}"
        print(line, flush=True)
