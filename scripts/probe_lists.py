import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import synth
S2 = 262144
c2 = hfz.Context(0, S2)
dev = c2.device
n = 1024
tr = synth.bb_traces(n, seed=44)
i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(dev)
lo, to, eo = i64(tr["launch_off"]), i64(tr["thread_off"]), i64(tr["ev_off"])
dims = torch.from_numpy(tr["dims"].view(np.int32)).to(dev)
sites = torch.from_numpy(tr["sites"].view(np.int32)).to(dev)
o = None; g = None
v, c = c2.new_virgin(), c2.new_edge_counts()
for it in range(3):
    o = c2.edge_record_batch_lists(lo, dims, to, eo, sites, n, cap=6144, out=o)
    v.zero_(); c.zero_()
    g = c2.feedback_batch_sparse(o["entries"], o["entry_off"], v, c, out=g)
torch.cuda.synchronize()
print("ok", int((g["admit"] != 0).sum()))
