"""Dev probe: throughput of K3 (havoc, config 4) and K1 (edge record, config 3) + K2 odd cases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_12485_b200 as hfz
from paper_2603_12485_b200 import api, synth

def timeit(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[1:])

ctx = hfz.Context(0, int(os.environ.get("EDGE_S", "65536")))
ctx.set_option("edge_flat", int(os.environ.get("EDGE_FLAT", "1")))
dev = ctx.device
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "havoc"):
    n = 16384
    data, off = synth.havoc_inputs(n, seed=45)
    d_in = torch.from_numpy(np.concatenate([data, np.zeros(16, np.uint8)])).to(dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    seeds = torch.from_numpy(api.u64_to_i64(np.arange(1000, 1000 + n, dtype=np.uint64))).to(dev)
    st = seeds.clone()
    res = {}
    res["o"] = ctx.havoc_batch(d_in, d_off, st)  # sizes the output buffers once (host sync)
    def run():
        st.copy_(seeds)
        res["o"] = ctx.havoc_batch(d_in, d_off, st, out=res["o"])  # the kernel alone
    ms = timeit(run)
    ob, oo, ol, dr = res["o"]
    tot = int(off[-1]) + int(ol.sum().item())
    print(f"K3 havoc: {n} seeds, {ms:.3f} ms -> {n/ms*1e3/1e6:.2f} M mutants/s, sum(in+out) {tot/ms/1e6:.1f} GB/s, mean draws {dr.float().mean().item():.1f}")
if what in ("all", "edge"):
    for n_exec in (int(os.environ.get("EDGE_N", "2048")),):
        t = time.time()
        tr = synth.bb_traces(n_exec, seed=44)
        print(f"generated traces for {n_exec} execs in {time.time()-t:.1f}s: {tr['sites'].size/n_exec:.0f} events/exec")
        i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(dev)
        lo, to, eo = i64(tr["launch_off"]), i64(tr["thread_off"]), i64(tr["ev_off"])
        dims = torch.from_numpy(tr["dims"].view(np.int32)).to(dev)
        sites = torch.from_numpy(tr["sites"].view(np.int32)).to(dev)
        raw = torch.zeros(n_exec * ctx.rec, dtype=torch.uint8, device=dev)
        res = {}
        def run():
            res["o"] = ctx.edge_record_batch(lo, dims, to, eo, sites, n_exec, raw=raw)
        ms = timeit(run, reps=3)
        ev = tr["sites"].size
        threads = int(tr["thread_off"][-1])
        byts = 4 * ev + 8 * threads + 4 * (ctx.S // 2) * n_exec
        import ctypes
        from paper_2603_12485_b200 import _lib
        L = _lib.lib if hasattr(_lib, "lib") else None
        if L is not None and hasattr(L, "hfz_dbg_edge_prof"):
            buf = (ctypes.c_ulonglong * 32)()
            L.hfz_dbg_edge_prof(buf, 1); run(); torch.cuda.synchronize(); L.hfz_dbg_edge_prof(buf, 1)
            names = ["pop", "setup", "coherent", "fast", "handover", "t.clear", "t.phase1", "t.rows", "t.phase2", "-", "owner idle", "barrier", "zero/flush", "-", "-", "kernel(cta)"]
            tot = buf[15] / 1.0
            for role in (0, 1):
                print(("owners    " if role == 0 else "non-owners") + " (16 warps, % of CTA time each warp): " + ", ".join(
                    f"{names[c]} {buf[role * 16 + c] / 16 / tot * 100:.1f}" for c in range(13) if names[c] != "-"))
        print(f"K1 edge record: {n_exec} execs, {ms:.3f} ms -> {n_exec/ms*1e3:.0f} execs/s, {ev/ms/1e6:.2f} G events/s, {byts/ms/1e6:.1f} GB/s algorithmic, bumps/exec {res['o'][1].float().mean().item():.0f}")
if what in ("all", "k2"):
    S = 65536
    for mode, n in (("iid", 16384), ("campaign", 1024), ("campaign", 4096)):
        gen = synth.maps_iid if mode == "iid" else synth.maps_campaign
        raw = torch.empty(n * ctx.rec, dtype=torch.uint8, device=dev)
        for i in range(0, n, 2048):
            m = min(2048, n - i)
            raw[i * ctx.rec:(i + m) * ctx.rec] = torch.from_numpy(gen(m, S, first=i)).to(dev)
        virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
        for warm in (False, True):
            if warm:
                ctx.feedback_batch(torch.from_numpy(gen(4096, S, first=1 << 20)).to(dev), virgin, counts)
            v0 = virgin.clone()
            res = {}
            def run():
                virgin.copy_(v0)
                res["o"] = ctx.feedback_batch(raw, virgin, counts, out=res.get("o"))
            ms = timeit(run, reps=3)
            adm = int((res["o"]["admit"] != 0).sum())
            print(f"K2 {mode} n={n} warm={warm}: {ms:.3f} ms -> {n/ms*1e3/1e6:.2f} M evals/s, {n*ctx.rec/ms/1e6:.0f} GB/s, admits {adm}")
    c2 = hfz.Context(0, 262144)
    n = 4096
    raw = torch.empty(n * c2.rec, dtype=torch.uint8, device=dev)
    for i in range(0, n, 512):
        raw[i * c2.rec:(i + 512) * c2.rec] = torch.from_numpy(synth.maps_campaign(512, 262144, first=i)).to(dev)
    virgin, counts = c2.new_virgin(), c2.new_edge_counts()
    c2.feedback_batch(torch.from_numpy(synth.maps_campaign(1024, 262144, first=1 << 20)).to(dev), virgin, counts)
    v0 = virgin.clone()
    res = {}
    def run2():
        virgin.copy_(v0)
        res["o"] = c2.feedback_batch(raw, virgin, counts, out=res.get("o"))
    ms = timeit(run2, reps=3)
    print(f"K2 262144-slot n={n}: {ms:.3f} ms -> {n/ms*1e3/1e6:.3f} M evals/s, {n*c2.rec/ms/1e6:.0f} GB/s, admits {int((res['o']['admit']!=0).sum())}")
