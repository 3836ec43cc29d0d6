"""Dev probe: the dense fold between 4,096 and 65,536 maps -- automatic path vs the fused step forced, with the
fused step's phase timestamps (us since the first CTA started)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth

dev = torch.device("cuda", 0)
S = 65536
ctx = hfz.Context(0, S)
rec = ctx.rec
NS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4096, 8192, 12288, 16384, 20480, 24576, 32768, 40960, 49152, 65536]
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


def timeit(n, state, reps=12):
    out = None
    ms = []
    for r in range(reps + 3):
        if state == "warm":
            vw.copy_(vw0); cw.copy_(cw0)
        else:
            vw.zero_(); cw.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = ctx.feedback_batch(raws[r & 1][: n * rec], vw, cw, out=out); e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ms.append(e0.elapsed_time(e1))
    return float(np.mean(ms)), float(np.min(ms))


for n in NS:
    row = [f"n={n:6d} ideal={n*rec/6541.5e6:.3f}"]
    ctx.set_option("scan_two_stage", -1); ctx.set_option("step_probe", 0)
    for state in ("warm", "cold"):
        m, mn = timeit(n, state)
        row.append(f"auto/{state} {m:.3f} ({mn:.3f})")
    if n * S <= 1 << 30:
        ctx.set_option("scan_two_stage", 1 << 40)
        for state in ("warm", "cold"):
            m, mn = timeit(n, state)
            row.append(f"fused/{state} {m:.3f} ({mn:.3f})")
        ctx.set_option("step_probe", 1)
        timeit(n, "warm", reps=1)
        t = [ctx.get_stat(f"step_t{k}") for k in range(1, 7)]
        cy = [ctx.get_stat(f"step_c{k}") for k in range(6)]
        row.append(f"phases us: compact {t[0]:.0f} scrub {t[1]:.0f} sync1 {t[2]:.0f} roles {t[3]:.0f} sync2 {t[4]:.0f} resolve {t[5]:.0f}; warp0 compact {cy[5]:.0f} items wait {cy[3]/max(cy[5],1):.0f} work {cy[4]/max(cy[5],1):.0f} cyc/item; map0 gather {cy[0]:.0f} chain {cy[1]:.0f} cyc / {cy[2]:.0f} entries")
    print(" | ".join(row), flush=True)
