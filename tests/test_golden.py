"""Committed golden vectors (tests/golden/, generated from the compiled reference by
oracle/make_golden.py): checked against the C restatement on CPU and against the CUDA path on
the GPU box, where /root/reference does not exist."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2603_12485_b200 import synth

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
S, H = 65536, 32768


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def feedback_inputs(name):
    if name == "iid_64":
        return synth.maps_iid(64, S, seed=42), 64
    if name == "campaign_256":
        return synth.maps_campaign(256, S, seed=43, p_extra=16, p_rare=16), 256
    return synth.maps_edge_cases(S)


def check_feedback(o, v, c, want):
    assert o["admit"].tolist() == want["admit"]
    assert [f"{x:016x}" for x in o["sig_full"].tolist()] == want["sig_full"]
    assert [f"{x:016x}" for x in o["sig_simple"].tolist()] == want["sig_simple"]
    assert o["nnz"].tolist() == want["nnz"]
    assert sha(o["classed"]) == want["classed_sha256"]
    assert sha(v) == want["virgin_sha256"] and c.tolist() == want["edge_counts"]


@pytest.mark.parametrize("name", ["iid_64", "campaign_256", "edge_cases"])
def test_feedback_golden_cpu(port, name):
    want = json.load(open(os.path.join(G, "feedback.json")))[name]
    raw, n = feedback_inputs(name)
    assert sha(raw) == want["raw_sha256"], "synthetic generator drifted: regenerate the fixtures"
    v, c = np.zeros(S, np.uint8), np.zeros(2, np.uint64)
    check_feedback(port.feedback_batch(raw, n, S, v, c, want_classed=True), v, c, want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["iid_64", "campaign_256", "edge_cases"])
def test_feedback_golden_gpu(ctx, name):
    import torch
    want = json.load(open(os.path.join(G, "feedback.json")))[name]
    raw, n = feedback_inputs(name)
    virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
    o = ctx.feedback_batch(torch.from_numpy(raw).to(ctx.device), virgin, counts, want_classed=True)
    ctx.synchronize()
    res = dict(admit=o["admit"].cpu().numpy(), sig_full=o["sig_full"].cpu().numpy().view(np.uint64),
               sig_simple=o["sig_simple"].cpu().numpy().view(np.uint64), nnz=o["nnz"].cpu().numpy().view(np.uint32),
               classed=o["classed"].cpu().numpy())
    check_feedback(res, virgin.cpu().numpy(), counts.cpu().numpy().view(np.uint64), want)


def test_mutators_golden_cpu(port):
    g = json.load(open(os.path.join(G, "mutators.json")))
    for h in g["havoc"]:
        out, st, dr = port.havoc(bytes.fromhex(h["input"]), h["seed"])
        assert (out.hex(), st, dr) == (h["output"], h["end_state"], h["draws"])
    for s in g["splice"]:
        out, st = port.splice(bytes.fromhex(s["a"]), bytes.fromhex(s["b"]), s["seed"])
        assert (out.hex(), st) == (s["output"], s["end_state"])
    for d in g["deterministic"]:
        ms = port.deterministic(bytes.fromhex(d["input"]))
        assert len(ms) == d["count"] and hashlib.sha256(b"".join(ms)).hexdigest() == d["sha256"]


@pytest.mark.gpu
def test_mutators_golden_gpu(ctx):
    import paper_2603_12485_b200 as hfz
    g = json.load(open(os.path.join(G, "mutators.json")))
    outs, ends, draws = hfz.havoc_batch([bytes.fromhex(h["input"]) for h in g["havoc"]], [h["seed"] for h in g["havoc"]])
    for h, o, e, d in zip(g["havoc"], outs, ends, draws):
        assert (o.hex(), e, d) == (h["output"], h["end_state"], h["draws"])
    for s in g["splice"]:
        assert hfz.splice_mutant(bytes.fromhex(s["a"]), bytes.fromhex(s["b"]), s["seed"]).hex() == s["output"]
    for d in g["deterministic"]:
        ms = hfz.deterministic_mutants(bytes.fromhex(d["input"]))
        assert len(ms) == d["count"] and hashlib.sha256(b"".join(ms)).hexdigest() == d["sha256"]
        assert [m.hex() for m in ms[:4]] == d["first"]


def edge_traces(g):
    a, b = g["recipe_a"], g["recipe_b"]
    ta = synth.bb_traces(a["n"], seed=a["seed"], grid=tuple(a["grid"]), block=tuple(a["block"]), n_launch=a["n_launch"])
    tb = synth.bb_traces(b["n"], seed=b["seed"], grid=tuple(b["grid"]), block=tuple(b["block"]), n_launch=b["n_launch"])
    return [(ta, a["n"]), (tb, b["n"])]


def check_edges(raws, evs, g):
    k = 0
    rec = synth.record_bytes(S)
    for raw, ev in zip(raws, evs):
        dev = raw.reshape(-1, rec)[:, H:].view(np.uint32)
        for e in range(dev.shape[0]):
            want = g["execs"][k]
            nzi = np.nonzero(dev[e])[0]
            assert nzi.tolist() == want["slots"] and dev[e][nzi].tolist() == want["counts"]
            assert int(ev[e]) == want["warp_events"]
            k += 1
    assert k == len(g["execs"])


def test_edge_record_golden_cpu(port):
    g = json.load(open(os.path.join(G, "edge_record.json")))
    raws, evs = [], []
    for tr, n in edge_traces(g):
        raw, ev = port.edge_record_batch(tr["launch_off"], tr["dims"], tr["thread_off"], tr["ev_off"], tr["sites"], n, S)
        raws.append(raw)
        evs.append(ev)
    check_edges(raws, evs, g)


@pytest.mark.gpu
def test_edge_record_golden_gpu(ctx):
    from tests.test_edge_record_gpu import run_gpu
    g = json.load(open(os.path.join(G, "edge_record.json")))
    raws, evs = [], []
    for tr, n in edge_traces(g):
        raw, ev = run_gpu(ctx, tr, n)
        raws.append(raw)
        evs.append(ev)
    check_edges(raws, evs, g)
