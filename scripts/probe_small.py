"""Dev probe: small-batch fold, legacy two-stage launches vs the fused cooperative step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth


def timeit(fn, pre, reps=30):
    for _ in range(3):
        pre(); fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    return float(np.mean(ms)), float(np.min(ms))


dev = torch.device("cuda", 0)
for S, ns in ((65536, (256, 1024, 2048, 4096, 8192, 12288, 16384)), (262144, (256, 1024, 2048, 4096))):
    ctx = hfz.Context(0, S)
    nmax = max(ns)
    rec = ctx.rec
    copies = 4 if nmax * rec * 4 < 12e9 else 2
    raws = []
    for b in range(copies):
        raw = torch.empty(nmax * rec, dtype=torch.uint8, device=dev)
        step = 2048 if S == 65536 else 512
        for i in range(0, nmax, step):
            raw[i * rec:(i + step) * rec] = torch.from_numpy(synth.maps_campaign(step, S, first=b * nmax + i)).to(dev)
        raws.append(raw)
    vw, cw = ctx.new_virgin(), ctx.new_edge_counts()
    ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(1024 if S > 65536 else 4096, S, first=1 << 24)).to(dev), vw, cw)
    vw0, cw0 = vw.clone(), cw.clone()
    for n in ns:
        row = [f"S={S} n={n:5d} ideal={n*rec/6544.3e6:.3f}ms"]
        for name, opts in (("legacy", dict(scan_two_stage=1 << 40, small_fused=0)), ("fused", dict(scan_two_stage=1 << 40, small_fused=1)),
                           ("auto", dict(scan_two_stage=-1, small_fused=1))):
            for k, v in opts.items():
                ctx.set_option(k, v)
            for state in ("warm", "cold"):
                st = {"i": 0, "o": None}
                def pre():
                    if state == "warm":
                        vw.copy_(vw0); cw.copy_(cw0)
                    else:
                        vw.zero_(); cw.zero_()
                    st["i"] += 1
                def fn():
                    st["o"] = ctx.feedback_batch(raws[st["i"] % copies][: n * rec], vw, cw, out=st["o"])
                l0 = ctx.launch_count
                mean, mn = timeit(fn, pre)
                row.append(f"{name}/{state} {mean:.3f} (min {mn:.3f}, {(ctx.launch_count-l0)/33:.0f} launches)")
        print(" | ".join(row), flush=True)
    ctx.close()
    del raws
