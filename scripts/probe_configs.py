#!/usr/bin/env python
"""One line per BASELINE.json config (device-resident, CUDA events, best of 3): the secondary
numbers quoted in DESIGN.md next to the headline of bench.py (configs[1])."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import api, synth


def best(fn, reps=3):
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])


dev = torch.device("cuda", 0)
PEAK = 6544.3

# configs[0]: 1,024 maps of 65,536 slots, cold virgin (the parity configuration)
S = 65536
ctx = hfz.Context(0, S)
raw = torch.from_numpy(synth.maps_campaign(1024, S)).to(dev)
v, c = ctx.new_virgin(), ctx.new_edge_counts()
def run0():
    v.zero_(); c.zero_(); ctx.feedback_batch(raw, v, c)
ms = best(run0)
print(f"configs[0] 1,024 maps x 64 KB, cold virgin: {ms:.3f} ms -> {1024/ms/1e3:.2f} M evals/s ({1024*ctx.rec/ms/1e6:.0f} GB/s)")
ctx.close()

# configs[2]: 262,144-slot maps from synthetic basic-block traces: edge record (K1) then the fold (K2)
S2 = 262144
n = int(os.environ.get("CFG2_EXECS", "1024"))
c2 = hfz.Context(0, S2)
t = time.time()
tr = synth.bb_traces(n, seed=44)
gen = time.time() - t
i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(dev)
lo, to, eo = i64(tr["launch_off"]), i64(tr["thread_off"]), i64(tr["ev_off"])
dims = torch.from_numpy(tr["dims"].view(np.int32)).to(dev)
sites = torch.from_numpy(tr["sites"].view(np.int32)).to(dev)
raw2 = torch.zeros(n * c2.rec, dtype=torch.uint8, device=dev)
ms_k1 = best(lambda: c2.edge_record_batch(lo, dims, to, eo, sites, n, raw=raw2))
v2, cc2 = c2.new_virgin(), c2.new_edge_counts()
def run2():
    v2.zero_(); cc2.zero_(); c2.feedback_batch(raw2, v2, cc2)
ms_k2 = best(run2)
ev = tr["sites"].size
print(f"configs[2] {n} execs, 262,144-slot maps, {ev/n:.0f} events/exec (traces generated in {gen:.0f} s): "
      f"edge record {ms_k1:.3f} ms ({n/ms_k1*1e3:.0f} execs/s, {ev/ms_k1/1e6:.1f} G events/s) + fold {ms_k2:.3f} ms "
      f"({n*c2.rec/ms_k2/1e6:.0f} GB/s) = {n/(ms_k1+ms_k2)*1e3:.0f} execs/s end to end on the device")
c2.close()

# configs[3]: havoc of 16,384 seeds of 1-4 KB
ctx = hfz.Context(0, S)
data, off = synth.havoc_inputs(16384, seed=45)
d_in = torch.from_numpy(np.concatenate([data, np.zeros(16, np.uint8)])).to(dev)
d_off = torch.from_numpy(off.view(np.int64)).to(dev)
seeds = torch.from_numpy(api.u64_to_i64(np.arange(1000, 1000 + 16384, dtype=np.uint64))).to(dev)
st = seeds.clone()
out = ctx.havoc_batch(d_in, d_off, st)
def run3():
    st.copy_(seeds); ctx.havoc_batch(d_in, d_off, st, out=out)
ms = best(run3, reps=5)
tot = int(off[-1]) + int(out[2].sum().item())
print(f"configs[3] havoc of 16,384 seeds (1-4 KB): {ms:.3f} ms -> {16384/ms/1e3:.1f} M mutants/s, {tot/ms/1e6:.0f} GB/s of in+out")

# configs[4] shape on ONE GPU: 8 simulated ranks x 8,192 execs (scan per rank, deltas concatenated, rank-ordered resolve)
R, per = 8, 8192
ctxs = [hfz.Context(0, S) for _ in range(R)]
raw = torch.empty(R * per * ctx.rec, dtype=torch.uint8, device=dev)
for i in range(0, R * per, 4096):
    raw[i * ctx.rec:(i + 4096) * ctx.rec] = torch.from_numpy(synth.maps_campaign(4096, S, first=i)).to(dev)
v0, c0 = ctx.new_virgin(), ctx.new_edge_counts()
ctx.feedback_batch(torch.from_numpy(synth.maps_campaign(4096, S, first=1 << 24)).to(dev), v0, c0)
shards = [raw[r * per * ctx.rec:(r + 1) * per * ctx.rec] for r in range(R)]
def run4():
    scans = [ctxs[r].feedback_scan(shards[r], v0) for r in range(R)]
    deltas = torch.cat([s["delta"] for s in scans])
    for r in range(R):
        ctxs[r].feedback_resolve(shards[r], v0.clone(), c0.clone(), deltas, R, r)
ms = best(run4)
print(f"configs[4] shape on one GPU: 8 simulated ranks x 8,192 execs, scan + delta exchange + rank-ordered resolve: "
      f"{ms:.3f} ms for 65,536 execs ({R*per/ms/1e3:.1f} M evals/s on one device; the 8-GPU number is bench.py --gpus 8)")
