"""Dev probe: lane-per-map scan with 256 / 512 / 1,024-byte rows (32 / 32 / 16 maps per warp) against the automatic dispatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

dev = torch.device("cuda", 0)
S = 65536
ctx = hfz.Context(0, S)
rec = ctx.rec
NS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8192, 10240, 12288, 14336, 16384, 20480, 24576, 28672, 32768, 40960, 49152, 65536]
nmax = max(NS)
raws = []
for b in range(2):
    raw = torch.empty(nmax * rec, dtype=torch.uint8, device=dev)
    for i in range(0, nmax, 2048):
        raw[i * rec:(i + 2048) * rec] = torch.from_numpy(synth.maps_campaign(2048, S, first=b * nmax + i)).to(dev)
    raws.append(raw)
vw, cw = ctx.new_virgin(), ctx.new_edge_counts()
ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(4096, S, first=1 << 24)).to(dev), vw, cw)
vw0, cw0 = vw.clone(), cw.clone()


def timeit(n, reps=12):
    out = None
    ms = []
    for r in range(reps + 3):
        vw.copy_(vw0); cw.copy_(cw0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = ctx.feedback_batch(raws[r & 1][: n * rec], vw, cw, out=out); e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ms.append(e0.elapsed_time(e1))
    return float(np.mean(ms))


for n in NS:
    row = [f"n={n:6d} ideal={n*rec/6541.5e6:.3f}"]
    for k in ("scan_small", "scan_pipe", "scan_two_stage"):
        ctx.set_option(k, -1)
    ctx.set_option("small_fused", 1); ctx.set_option("scan_row", 0)
    row.append(f"auto {timeit(n):.3f}")
    ctx.set_option("scan_small", 0); ctx.set_option("scan_pipe", 0); ctx.set_option("scan_two_stage", 0); ctx.set_option("small_fused", 0)
    for r in (256, 512, 1024):
        ctx.set_option("scan_row", r)
        row.append(f"row{r} {timeit(n):.3f}")
    print(" | ".join(row), flush=True)
