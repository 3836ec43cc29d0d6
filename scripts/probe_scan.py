"""Dev probe: the dense fold at a few batch sizes, warm / cold / iid (for comparing builds of libhfz.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

dev = torch.device("cuda", 0)
S = 65536
ctx = hfz.Context(0, S)
rec = ctx.rec
NS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [12288, 16384, 32768, 65536]
nmax = max(NS)
raw = torch.empty(nmax * rec, dtype=torch.uint8, device=dev)
for i in range(0, nmax, 2048):
    raw[i * rec:(i + 2048) * rec] = torch.from_numpy(synth.maps_campaign(2048, S, first=i)).to(dev)
iid = torch.empty(nmax * rec, dtype=torch.uint8, device=dev)
for i in range(0, nmax, 2048):
    iid[i * rec:(i + 2048) * rec] = torch.from_numpy(synth.maps_iid(2048, S, first=i)).to(dev)
vw, cw = ctx.new_virgin(), ctx.new_edge_counts()
ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(4096, S, first=1 << 24)).to(dev), vw, cw)
vw0, cw0 = vw.clone(), cw.clone()
vi, ci = ctx.new_virgin(), ctx.new_edge_counts()
ctx.feedback_batch(torch.from_numpy(synth.maps_iid(4096, S, first=1 << 24)).to(dev), vi, ci)
vi0 = vi.clone()


def timeit(buf, n, v0, reps=20):
    out = None
    ms = []
    for r in range(reps + 3):
        if v0 is None:
            vw.zero_()
        else:
            vw.copy_(v0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = ctx.feedback_batch(buf[: n * rec], vw, cw, out=out); e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ms.append(e0.elapsed_time(e1))
    return float(np.mean(ms)), float(np.min(ms))


for n in NS:
    w, c, i = timeit(raw, n, vw0), timeit(raw, n, None), timeit(iid, n, vi0)
    print(f"n={n:6d} ideal={n*rec/6541.5e6:.3f} | warm {w[0]:.3f} ({w[1]:.3f}) | cold {c[0]:.3f} ({c[1]:.3f}) | iid {i[0]:.3f} ({i[1]:.3f})", flush=True)
