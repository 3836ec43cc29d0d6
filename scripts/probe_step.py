"""Dev probe: phase timestamps inside the fused small step (us since the first CTA started)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth
dev = torch.device("cuda", 0)
for S, ns in ((65536, (256, 1024, 4096)), (262144, (256, 1024))):
    ctx = hfz.Context(0, S)
    ctx.set_option("step_probe", 1)
    ctx.set_option("scan_two_stage", 1 << 40)
    for n in ns:
        raw = torch.from_numpy(synth.maps_campaign(n, S)).to(dev)
        v, c = ctx.new_virgin(), ctx.new_edge_counts()
        ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(512, S, first=1 << 24)).to(dev), v, c)
        v0 = v.clone()
        for rep in range(3):
            v.copy_(v0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ctx.feedback_batch(raw, v, c); e1.record(); torch.cuda.synchronize()
            t = [ctx.get_stat(f"step_t{k}") for k in range(1, 7)]
            cy = [ctx.get_stat(f"step_c{k}") for k in range(6)]
        print(f"S={S} n={n}: event {e0.elapsed_time(e1)*1e3:.0f} us | compact {t[0]:.0f} scrub {t[1]:.0f} sync1 {t[2]:.0f} roles {t[3]:.0f} sync2 {t[4]:.0f} resolve {t[5]:.0f} | map 0: gather {cy[0]:.0f} cyc, chain {cy[1]:.0f} cyc for {cy[2]:.0f} entries = {cy[1]/max(cy[2],1):.1f} cyc/entry | warp 0 compact: {cy[5]:.0f} items, wait {cy[3]/max(cy[5],1):.0f} + work {cy[4]/max(cy[5],1):.0f} cyc/item", flush=True)
    ctx.close()
