#!/usr/bin/env python
"""Generate tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref, compiled from
/root/reference by oracle/build_ref.sh).  Run in the build container only; the fixtures are
committed so that the GPU box (which has no /root/reference) can check against them.

    python oracle/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402
from paper_2603_12485_b200 import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
os.makedirs(OUT, exist_ok=True)
S = 65536
ref = pyoracle.Ref(S)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --- feedback: inputs are regenerated from seeds by synth (deterministic); outputs stored
fb = {}
for name, raw, n in (("iid_64", synth.maps_iid(64, S, seed=42), 64),
                     ("campaign_256", synth.maps_campaign(256, S, seed=43, p_extra=16, p_rare=16), 256),
                     ("edge_cases", *synth.maps_edge_cases(S))):
    v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    o = ref.feedback_batch(raw, n, S, v, c, want_classed=True)
    fb[name] = dict(n=n, raw_sha256=sha(raw), admit=o["admit"].tolist(),
                    sig_full=[f"{x:016x}" for x in o["sig_full"].tolist()],
                    sig_simple=[f"{x:016x}" for x in o["sig_simple"].tolist()], nnz=o["nnz"].tolist(),
                    classed_sha256=sha(o["classed"]), virgin_sha256=sha(v), edge_counts=c.tolist(),
                    virgin_nonzero=int(np.count_nonzero(v)))
json.dump(fb, open(os.path.join(OUT, "feedback.json"), "w"), indent=0)

# --- havoc / splice / deterministic: explicit byte strings
rng = np.random.default_rng(2026)
hv = []
for i in range(96):
    ln = [0, 1, 2, 3, 4, 5, 8, 16, 33, 64, 100, 257][i % 12] if i < 72 else int(rng.integers(200, 1500))
    data = rng.integers(0, 256, ln, dtype=np.uint8).tobytes()
    seed = int(rng.integers(0, 2 ** 63))
    out, st, draws = ref.havoc(data, seed)
    hv.append(dict(input=data.hex(), seed=seed, output=out.hex(), end_state=st, draws=draws))
sp = []
for i in range(32):
    a = rng.integers(0, 256, int(rng.integers(0, 40)), dtype=np.uint8).tobytes()
    b = rng.integers(0, 256, int(rng.integers(0, 40)), dtype=np.uint8).tobytes()
    seed = int(rng.integers(0, 2 ** 63))
    out, st = ref.splice(a, b, seed)
    sp.append(dict(a=a.hex(), b=b.hex(), seed=seed, output=out.hex(), end_state=st))
det = []
for ln in (1, 2, 3, 4, 8, 33):
    d = rng.integers(0, 256, ln, dtype=np.uint8).tobytes()
    ms = ref.deterministic(d)
    det.append(dict(input=d.hex(), count=len(ms), sha256=hashlib.sha256(b"".join(ms)).hexdigest(),
                    first=[m.hex() for m in ms[:4]]))
json.dump(dict(havoc=hv, splice=sp, deterministic=det), open(os.path.join(OUT, "mutators.json"), "w"), indent=0)

# --- edge record through the real runtime: traces regenerated from seeds, sparse counters stored
er = []
tr = synth.bb_traces(4, seed=44, grid=(2, 1, 1), block=(100, 1, 1), n_launch=3)
for e in range(4):
    l0, l1 = int(tr["launch_off"][e]), int(tr["launch_off"][e + 1])
    t0 = int(tr["thread_off"][l0])
    c, n = ref.edge_record_exec(tr["dims"][l0:l1], tr["ev_off"][t0:], tr["sites"])
    nzi = np.nonzero(c)[0]
    er.append(dict(slots=nzi.tolist(), counts=c[nzi].tolist(), warp_events=n))
tr3 = synth.bb_traces(2, seed=9, grid=(2, 3, 2), block=(4, 2, 3), n_launch=2)
for e in range(2):
    l0, l1 = int(tr3["launch_off"][e]), int(tr3["launch_off"][e + 1])
    t0 = int(tr3["thread_off"][l0])
    c, n = ref.edge_record_exec(tr3["dims"][l0:l1], tr3["ev_off"][t0:], tr3["sites"])
    nzi = np.nonzero(c)[0]
    er.append(dict(slots=nzi.tolist(), counts=c[nzi].tolist(), warp_events=n))
json.dump(dict(recipe_a=dict(n=4, seed=44, grid=[2, 1, 1], block=[100, 1, 1], n_launch=3),
               recipe_b=dict(n=2, seed=9, grid=[2, 3, 2], block=[4, 2, 3], n_launch=2), execs=er),
          open(os.path.join(OUT, "edge_record.json"), "w"), indent=0)
print("golden fixtures written to", OUT, {f: os.path.getsize(os.path.join(OUT, f)) for f in os.listdir(OUT)})
