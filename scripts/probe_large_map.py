import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth
S2 = 262144
c2 = hfz.Context(0, S2)
for n in (1024, 4096):
    raw = torch.empty(n * c2.rec, dtype=torch.uint8, device=c2.device)
    for i in range(0, n, 512):
        raw[i * c2.rec:(i + 512) * c2.rec] = torch.from_numpy(synth.maps_campaign(512, S2, first=i)).to(c2.device)
    virgin, counts = c2.new_virgin(), c2.new_edge_counts()
    c2.feedback_batch(raw, virgin, counts)
    v0 = virgin.clone()
    for name, opts in (("lane", dict(scan_small=0, scan_pipe=0, scan_two_stage=0)), ("pipe", dict(scan_small=0, scan_pipe=1 << 20, scan_two_stage=0)),
                       ("two", dict(scan_small=0, scan_pipe=0, scan_two_stage=1 << 40)), ("auto", dict(scan_small=-1, scan_pipe=-1, scan_two_stage=-1))):
        for k, v in opts.items():
            c2.set_option(k, v)
        ts = []
        for r in range(5):
            virgin.copy_(v0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); c2.feedback_batch(raw, virgin, counts); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"S=262144 n={n} {name}: {min(ts[1:]):.3f} ms (ideal {n*c2.rec/6544.7e6:.3f})", flush=True)
