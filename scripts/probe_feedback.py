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
ap.add_argument("--mode", default="campaign")
ap.add_argument("--variants", default="1,2,3,4,5")
ap.add_argument("--warps", default="0")
ap.add_argument("--reps", type=int, default=5)
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
for var in [int(x) for x in a.variants.split(",")]:
    for w in [int(x) for x in a.warps.split(",")]:
        ctx.set_option("scan_variant", var)
        ctx.set_option("scan_warps", w)
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
        print(f"variant {var} warps {w:2d}: {ms:8.3f} ms  {a.n/ms*1e3/1e6:7.3f} M evals/s  "
              f"{a.n*rec/ms/1e6:8.1f} GB/s  admits {cand}", flush=True)
