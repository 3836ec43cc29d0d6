#!/usr/bin/env python
"""Headline benchmark: coverage-map evals/sec of the fused feedback step (BASELINE.json).

    python bench.py --gpus N --steps K --warmup W [--impl reference]

A "step" is one pass of the hot path (classify + has_new_bits + 2 signatures + virgin fold)
over one batch of synthetic raw maps: configs[1] of BASELINE.json, a 65,536-exec batch of
64 KB (65,536-slot) maps per GPU, ~2 % density, campaign-like novelty, virgin pre-warmed with
4,096 maps.  N > 1 (launched by torchrun, one rank per GPU) shards the campaign batch
(N x 65,536 execs), allgathers the per-rank novelty deltas over NCCL and merges in rank order
("scaling": "weak").  Prints ONE JSON line on rank 0.

At N = 1 the same line also carries the other named configs of BASELINE.json, each with its own
kernel time (CUDA events), algorithmic bytes, roofline fraction and CPU baseline, and each
oracle-checked at its stated size inside the run (a mismatch aborts without printing a number):
    config0_small_batch   configs[0]  1,024 maps of 65,536 slots (cold = the parity case, and warm)
    k1_edge_record        configs[2]  trace recipe, edge record alone into 65,536-slot maps
    config2_large_map     configs[2]  262,144-slot maps from traces: edge record -> fused fold
    k3_havoc              configs[3]  havoc of 16,384 seeds of 1-4 KB
"""
import argparse
import hashlib
import importlib.util
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

S = 65536
REC = (S // 2) * 5
S_LARGE = 262144
REC_LARGE = (S_LARGE // 2) * 5
METRIC = "coverage_map_evals_per_sec"
UNIT = "evals/s"

_synth = None


def synth():
    """The workload generator, loaded WITHOUT importing the package (whose __init__ dlopens
    libhfz.so): the reference arm must run on a box that has no CUDA library at all."""
    global _synth
    if _synth is None:
        spec = importlib.util.spec_from_file_location(
            "hfz_bench_synth", os.path.join(ROOT, "paper_2603_12485_b200", "synth.py"))
        _synth = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(_synth)
    return _synth


def make_maps(n, first, mode, slots=S):
    gen = synth().maps_campaign if mode == "campaign" else synth().maps_iid
    return gen(n, slots, first=first)


def workload_name(args):
    return (f"BASELINE.json configs[1]: {args.execs}-exec batch of 64 KB (65,536-slot) maps per GPU, "
            f"fused classify+has_new_bits+signatures, {args.mode}-like novelty, virgin pre-warmed with 4,096 maps")


def base_config(args, world):
    """The workload description: identical in both arms (the driver compares them)."""
    n = args.execs
    return {"workload": workload_name(args), "map_slots": S, "bytes_per_eval": REC, "execs_per_gpu": n,
            "global_execs_per_step": world * n, "density": 0.02, "mode": args.mode,
            "cpu_sample_execs": args.cpu_sample,
            "l2_policy": (f"inputs larger than L2 ({n * REC / 1e9:.1f} GB per GPU per step)" if n * REC > 512e6
                          else f"inputs of {n * REC / 1e6:.0f} MB per GPU may stay L2-resident (not a bench configuration)"),
            "parallelism": f"exec-sharded x{world}"}


def hbm_peak():
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        return float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU legs
# Every CPU leg runs the reference's own implementation (oracle/_ref, the unmodified sources
# compiled by oracle/build_ref.sh) when that build exists, else the plain-C restatement, on all
# host threads; ctypes releases the GIL, so one foreign call per Python thread runs in parallel.

def run_replicas(work, threads, min_seconds, reps_cap=1 << 30):
    """work(i) -> units done by one call on thread i; every thread repeats it until min_seconds
    have passed.  Returns (units/s, total reps, seconds)."""
    done = [0] * threads
    units = [0] * threads
    stop_at = [None]

    def worker(i):
        reps = 0
        while True:
            units[i] += work(i)
            reps += 1
            if reps >= reps_cap or time.perf_counter() >= stop_at[0]:
                break
        done[i] = reps

    t0 = time.perf_counter()
    stop_at[0] = t0 + min_seconds
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return sum(units) / dt, sum(done), dt


def cpu_feedback_rate(raw_sample, n_sample, v0, threads, min_seconds, reps_cap=64, slots=S):
    """Reference CPU path (classify_trace + 2x trace_signature + has_new_bits, engine.cpp:471-478)
    on `threads` host threads, each folding the whole sample as an independent replica with a
    private copy of the start virgin map.  Returns (evals/s, kind, reps, seconds)."""
    from oracle import pyoracle
    if pyoracle.Ref.available(slots):
        ck = pyoracle.Ref(slots)
        h = ck.maps_create(raw_sample, n_sample)  # CoverageMap objects, outside the timed region

        def work(i):
            ck.feedback_run(h, 0, n_sample, v0.copy(), np.zeros(2, np.uint64))
            return n_sample
    else:
        ck = pyoracle.Port()
        h = None
        adm = [np.zeros(n_sample, np.uint8) for _ in range(threads)]
        sf = [np.zeros(n_sample, np.uint64) for _ in range(threads)]
        ss = [np.zeros(n_sample, np.uint64) for _ in range(threads)]
        nz = [np.zeros(n_sample, np.uint32) for _ in range(threads)]

        def work(i):
            ck._feedback(raw_sample, n_sample, slots, v0.copy(), np.zeros(2, np.uint64), None, adm[i], sf[i], ss[i], nz[i])
            return n_sample

    rate, reps, dt = run_replicas(work, threads, min_seconds, reps_cap)
    if h is not None:
        ck.maps_free(h)
    return rate, ck.kind, reps, dt


def cpu_havoc_rate(data, off, ooff, seeds, threads, min_seconds):
    """havoc_mutant (src/engine.cpp:119-193): thread i mutates its own contiguous range of the
    seed set, over and over.  Returns (mutants/s, kind, reps, seconds)."""
    from oracle import pyoracle
    ck = pyoracle.best_checker(S)
    if ck.kind == "reference" and not ck.has_engine:
        ck = pyoracle.Port()
    n = off.size - 1
    out = np.zeros(int(ooff[-1]) + 64, np.uint8)
    olen = np.zeros(n, np.uint64)
    per = (n + threads - 1) // threads
    st = [seeds.copy() for _ in range(threads)]

    def work(i):
        a, b = min(n, i * per), min(n, (i + 1) * per)
        if b > a:
            st[i][a:b] = seeds[a:b]
            ck.havoc_range(data, off, a, b - a, st[i], out, ooff, olen)
        return b - a

    rate, reps, dt = run_replicas(work, threads, min_seconds)
    return rate, ck.kind, reps, dt


def cpu_edge_rate(tr, slots, threads, execs_per_thread, min_seconds):
    """Edge record through the reference runtime (hdvm::execute on a lambda-replay target, as
    tests/test_hdvm.cpp:66-85 builds them): thread i replays execs [i*k, (i+1)*k) of the trace
    batch.  Returns (execs/s, kind, reps, seconds, execs in the sample)."""
    from oracle import pyoracle
    ck = pyoracle.best_checker(slots)
    n = tr["launch_off"].size - 1
    k = max(1, min(execs_per_thread, n // threads))
    rec = (slots // 2) * 5
    raw = np.zeros(threads * k * rec, np.uint8)
    ev = np.zeros(threads * k, np.uint64)

    def work(i):
        ck.edge_record_range(tr, i * k, k, slots, raw, ev)
        return k

    rate, reps, dt = run_replicas(work, threads, min_seconds)
    return rate, ck.kind, reps, dt, threads * k


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on this box's host cores.  Imports
    nothing of the product (no libhfz.so): numpy, the workload generator file and oracle/ only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sample = args.cpu_sample
    raw = make_maps(n_sample, 0, args.mode)
    warm = make_maps(4096, 1 << 24, args.mode)
    from oracle import pyoracle
    ck = pyoracle.best_checker(S)
    v0 = np.zeros(S, np.uint8)
    ck.feedback_batch(warm, 4096, S, v0, np.zeros(2, np.uint64))
    for _ in range(args.warmup):
        cpu_feedback_rate(raw, n_sample, v0, threads, 0.0, reps_cap=1)
    rates, secs = [], 0.0
    kind = "port"
    for _ in range(args.steps):
        r, kind, reps, dt = cpu_feedback_rate(raw, n_sample, v0, threads, args.cpu_seconds / max(1, args.steps))
        rates.append(r)
        secs += dt
    value = float(np.mean(rates))
    sample = (f"first {n_sample} maps of the workload per replica, {threads} independent replicas "
              f"(private pre-warmed virgin), each step ~{args.cpu_seconds / max(1, args.steps):.1f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / max(1, args.steps) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32->u64", "data": "synthetic",
        "config": base_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm helpers
def sparse_lists_from_device(raw, n, dev):
    """Touched-slot lists of the first n records of `raw` (device tensor): pinned host tensors
    (entries (N, 2) int32, entry_off (n+1) int64).  The pairs of an exec are put in a random order.
    Data preparation, outside every timed region."""
    import torch
    H = S // 2
    ents, counts = [], []
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    for i in range(0, n, 2048):
        m = min(2048, n - i)
        rec = raw[i * REC:(i + m) * REC].view(m, REC)
        host = rec[:, :H]
        devh = rec[:, H:].contiguous().view(torch.int32)
        hr, hc = torch.nonzero(host, as_tuple=True)
        dr, dc = torch.nonzero(devh, as_tuple=True)
        rows = torch.cat([hr, dr])
        slots = torch.cat([hc, dc + H]).to(torch.int32)
        cnts = torch.cat([host[hr, hc].to(torch.int32), devh[dr, dc]])
        key = (rows << 32) | torch.randint(0, 1 << 31, rows.shape, device=dev, generator=g)
        order = torch.argsort(key)
        ents.append(torch.stack([slots[order], cnts[order]], dim=1).cpu())
        counts.append(torch.bincount(rows, minlength=m).cpu())
    total = sum(int(e.shape[0]) for e in ents)
    ent = torch.empty((total, 2), dtype=torch.int32, pin_memory=True)
    off = torch.zeros(n + 1, dtype=torch.int64, pin_memory=True)
    p = 0
    for e in ents:
        ent[p:p + e.shape[0]] = e
        p += e.shape[0]
    off[1:] = torch.cumsum(torch.cat(counts), 0)
    return ent, off


def compact_lists(ent, off):
    """8-byte pairs -> the 4-byte list form: compact words slot | count << 16 for counts below
    65,536 plus wide pairs for the rest (pinned host tensors; data preparation)."""
    import torch
    n = off.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n), off[1:] - off[:-1])
    cnt = ent[:, 1]
    big = (cnt < 0) | (cnt >= 65536)          # int32 view of u32 counts
    small = ~big
    comp = torch.empty(int(small.sum()), dtype=torch.int32, pin_memory=True)
    comp.copy_(ent[small, 0] | (ent[small, 1] << 16))
    wide = torch.empty((int(big.sum()), 2), dtype=torch.int32, pin_memory=True)
    wide.copy_(ent[big])
    coff = torch.zeros(n + 1, dtype=torch.int64, pin_memory=True)
    woff = torch.zeros(n + 1, dtype=torch.int64, pin_memory=True)
    coff[1:] = torch.cumsum(torch.bincount(rows[small], minlength=n), 0)
    woff[1:] = torch.cumsum(torch.bincount(rows[big], minlength=n), 0)
    return comp, coff, wide, woff


def packed_lists(ent, off):
    """8-byte pairs -> the packed list form of hfz_feedback_batch_packed_host: host half at 3 bytes per slot (slot lo,
    slot hi, count; every exec padded with zero entries to a multiple of four), device half at 4 bytes per slot
    ((slot - H) | min(count, 65536) << 15).  Pinned host tensors; data preparation."""
    import torch
    H = S // 2
    n = off.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n), off[1:] - off[:-1])
    slot, cnt = ent[:, 0], ent[:, 1]  # int32 views of u32 values
    is_host = slot < H
    nh = torch.bincount(rows[is_host], minlength=n)
    hoff = torch.zeros(n + 1, dtype=torch.int64, pin_memory=True)
    hoff[1:] = torch.cumsum((nh + 3) // 4 * 4, 0)
    hrows = rows[is_host]
    within = torch.arange(hrows.numel()) - (torch.cumsum(nh, 0) - nh)[hrows]
    dst = hoff[:-1][hrows] + within
    host3 = torch.zeros((int(hoff[-1]), 3), dtype=torch.uint8, pin_memory=True)
    hs, hc = slot[is_host], cnt[is_host]
    host3[dst, 0] = (hs & 0xFF).to(torch.uint8)
    host3[dst, 1] = (hs >> 8).to(torch.uint8)
    host3[dst, 2] = hc.to(torch.uint8)
    ds = (slot[~is_host] - H).to(torch.int64)
    dc = cnt[~is_host].to(torch.int64)
    dc = torch.where((dc < 0) | (dc > 65536), torch.full_like(dc, 65536), dc)
    w = ds | (dc << 15)
    w = torch.where(w >= (1 << 31), w - (1 << 32), w)  # the u32 bit pattern as int32
    dev17 = torch.empty(w.numel(), dtype=torch.int32, pin_memory=True)
    dev17.copy_(w.to(torch.int32))
    doff = torch.zeros(n + 1, dtype=torch.int64, pin_memory=True)
    doff[1:] = torch.cumsum(torch.bincount(rows[~is_host], minlength=n), 0)
    return host3.view(-1), hoff, dev17, doff


def fail(msg):
    raise SystemExit(f"bench.py: {msg} -- refusing to report a number")


class GpuTimer:
    """CUDA-event timing of fn() alone on torch's current stream (the stream the hfz context
    launches on); pre() -- state reset, L2 flush -- runs before every iteration, outside the bracket."""

    def __init__(self, dev):
        import torch
        self.torch = torch
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > the 126 MB L2

    def flush_l2(self):
        self.flush_buf.add_(1)

    def run(self, fn, iters, warmup=3, pre=None):
        torch = self.torch
        for _ in range(warmup):
            if pre:
                pre()
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(iters):
            if pre:
                pre()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
        return {"mean": float(np.mean(ms)), "min": float(np.min(ms)), "median": float(np.median(ms)), "iters": iters}


def roof(bytes_per_launch, ms, peak, peak_src, kernel, note=None):
    achieved = bytes_per_launch / (ms / 1e3) / 1e9
    r = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": None, "algorithmic_bytes_per_launch": int(bytes_per_launch), "kernel_ms_per_launch": ms,
         "peak_source": peak_src}
    if note:
        r["note"] = note
    return r


def u64dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(dev)


def traces_to_device(tr, dev):
    import torch
    return dict(launch_off=u64dev(tr["launch_off"], dev), thread_off=u64dev(tr["thread_off"], dev),
                ev_off=u64dev(tr["ev_off"], dev),
                dims=torch.from_numpy(np.ascontiguousarray(tr["dims"], np.uint32).view(np.int32)).to(dev),
                sites=torch.from_numpy(np.ascontiguousarray(tr["sites"], np.uint32).view(np.int32)).to(dev))


def trace_prefix(tr, n):
    """The first n execs of a trace batch (views; offsets are absolute, so no rebasing)."""
    nl = int(tr["launch_off"][n])
    nt = int(tr["thread_off"][nl])
    ne = int(tr["ev_off"][nt])
    return dict(launch_off=tr["launch_off"][:n + 1], dims=tr["dims"][:nl], thread_off=tr["thread_off"][:nl + 1],
                ev_off=tr["ev_off"][:nt + 1], sites=tr["sites"][:ne])


# --------------------------------------------------------------------------- the other named configs (N = 1)
def bench_config0(hfz, dev, timer, peak, peak_src, args, threads):
    """configs[0]: 1,024 maps of 65,536 slots, single rank.  Cold virgin = the parity configuration
    (every output compared with the oracle, all three Admit codes occur); warm = the steady state."""
    import torch
    from oracle import pyoracle
    n = 1024
    ctx = hfz.Context(dev.index, S)
    # four distinct batches, rotated, so no iteration finds its 168 MB input in the 126 MB L2
    hosts = [make_maps(n, b * n, "campaign") for b in range(4)]
    raws = [torch.from_numpy(h).to(dev) for h in hosts]
    virgin, counts = ctx.new_virgin(), ctx.new_edge_counts()
    # parity, cold: classed maps, Admit codes in order, both signatures, nnz, final virgin, counters
    ck = pyoracle.best_checker(S)
    out = ctx.feedback_batch(raws[0], virgin, counts, want_classed=True)
    torch.cuda.synchronize()
    v = np.zeros(S, np.uint8)
    c = np.zeros(2, np.uint64)
    want = ck.feedback_batch(hosts[0], n, S, v, c, want_classed=True)
    ok = (np.array_equal(out["admit"].cpu().numpy(), want["admit"])
          and np.array_equal(out["sig_full"].cpu().numpy().view(np.uint64), want["sig_full"])
          and np.array_equal(out["sig_simple"].cpu().numpy().view(np.uint64), want["sig_simple"])
          and np.array_equal(out["nnz"].cpu().numpy().view(np.uint32), want["nnz"])
          and np.array_equal(out["classed"].cpu().numpy(), want["classed"])
          and np.array_equal(virgin.cpu().numpy(), v)
          and np.array_equal(counts.cpu().numpy().view(np.uint64), c))
    if not ok:
        fail("configs[0] (1,024 maps, cold virgin): GPU results differ from the oracle")
    admits_cold = np.bincount(want["admit"], minlength=3).tolist()
    del out
    # warm state: the virgin after 4,096 other maps
    vw, cw = ctx.new_virgin(), ctx.new_edge_counts()
    ctx.feedback_batch(torch.from_numpy(make_maps(4096, 1 << 24, "campaign")).to(dev), vw, cw)
    vw0, cw0 = vw.clone(), cw.clone()
    res = {"o": None, "i": 0}

    def pre_cold():
        virgin.zero_()
        counts.zero_()
        res["i"] += 1

    def run_cold():
        res["o"] = ctx.feedback_batch(raws[res["i"] % 4], virgin, counts, out=res["o"])

    def pre_warm():
        vw.copy_(vw0)
        cw.copy_(cw0)
        res["i"] += 1

    def run_warm():
        res["o"] = ctx.feedback_batch(raws[res["i"] % 4], vw, cw, out=res["o"])

    l0 = ctx.launch_count
    t_warm = timer.run(run_warm, 40, pre=pre_warm)
    per_step = (ctx.launch_count - l0) / 43.0
    t_cold = timer.run(run_cold, 40, pre=pre_cold)
    byts = n * REC
    cpu = None
    if not args.no_cpu:
        rate, kind, reps, dt = cpu_feedback_rate(hosts[0], n, np.zeros(S, np.uint8), threads, min(4.0, args.cpu_seconds))
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"the 1,024 maps per replica from a cold virgin, {threads} independent replicas, {reps} folds in {dt:.1f} s"}
    ctx.close()
    return {"config": "BASELINE.json configs[0]: 1,024 synthetic 64 KB maps (~2 % density), classify + has_new_bits + signatures, single rank",
            "value": n / (t_warm["mean"] / 1e3), "unit": UNIT, "ms_per_step": t_warm["mean"], "ms_per_step_min": t_warm["min"],
            "state": "virgin pre-warmed with 4,096 maps (steady state)",
            "cold": {"value": n / (t_cold["mean"] / 1e3), "unit": UNIT, "ms_per_step": t_cold["mean"], "ms_per_step_min": t_cold["min"],
                     "admit_histogram": admits_cold,
                     "state": "empty virgin: every map is a candidate (the parity configuration)"},
            "iters": t_warm["iters"], "launches_per_step": per_step,
            "roofline": roof(byts, t_warm["mean"], peak, peak_src, "whole step (scan + resolve + merge launches)",
                             "latency-bound at this size: 168 MB is 26 us of HBM time"),
            "frac": byts / (t_warm["mean"] / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu,
            "parity_checked": "all 1,024 execs from a cold virgin: classed maps, Admit codes, both signatures, nnz, final virgin, both edge counters",
            "l2_policy": "four distinct 168 MB batches rotated: no iteration finds its input in L2"}


def bench_havoc(hfz, dev, timer, peak, peak_src, args, threads):
    """configs[3]: batched havoc of 16,384 seeds of 1-4 KB, per-slot Rng(1000 + j) (the Python-API
    semantics of bindings.cpp:220-223), byte-exact against havoc_mutant on EVERY slot."""
    import torch
    from oracle import pyoracle
    from paper_2603_12485_b200 import api
    n = 16384
    ctx = hfz.Context(dev.index, S)
    data, off = synth().havoc_inputs(n, seed=45)
    d_in = torch.from_numpy(np.concatenate([data, np.zeros(16, np.uint8)])).to(dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    seeds_np = np.arange(1000, 1000 + n, dtype=np.uint64)
    seeds = torch.from_numpy(api.u64_to_i64(seeds_np)).to(dev)
    st = seeds.clone()
    out = ctx.havoc_batch(d_in, d_off, st)  # sizes the output buffers once
    torch.cuda.synchronize()
    ob, oo, ol, dr = out
    # parity on all 16,384 slots: bytes, length, end state, draw count
    ck = pyoracle.best_checker(S)
    if ck.kind == "reference" and not ck.has_engine:
        ck = pyoracle.Port()
    ooff = oo.cpu().numpy().view(np.uint64)
    want_out = np.zeros(int(ooff[-1]) + 64, np.uint8)
    want_len = np.zeros(n, np.uint64)
    want_st = seeds_np.copy()
    per = (n + threads - 1) // threads
    ths = [threading.Thread(target=ck.havoc_range, args=(data, off, a, min(n, a + per) - a, want_st, want_out, ooff, want_len))
           for a in range(0, n, per)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    got_out = ob.cpu().numpy()
    got_len = ol.cpu().numpy().view(np.uint64)
    got_st = st.cpu().numpy().view(np.uint64)
    got_draws = dr.cpu().numpy().view(np.uint32).astype(np.uint64)
    gamma_inv = pow(0x9E3779B97F4A7C15, -1, 1 << 64)
    with np.errstate(over="ignore"):
        want_draws = (want_st - seeds_np) * np.uint64(gamma_inv)
    ok = np.array_equal(got_len, want_len) and np.array_equal(got_st, want_st) and np.array_equal(got_draws, want_draws)
    if ok:
        for j in range(n):
            a, L = int(ooff[j]), int(want_len[j])
            if not np.array_equal(got_out[a:a + L], want_out[a:a + L]):
                ok = False
                break
    if not ok:
        fail("configs[3] (havoc of 16,384 seeds): GPU mutants differ from the reference's havoc_mutant")

    def pre():
        st.copy_(seeds)
        timer.flush_l2()

    t = timer.run(lambda: ctx.havoc_batch(d_in, d_off, st, out=out), 20, pre=pre)
    byts = int(off[-1]) + int(want_len.sum())
    cpu = None
    if not args.no_cpu:
        rate, kind, reps, dt = cpu_havoc_rate(data, off, ooff, seeds_np, threads, min(4.0, args.cpu_seconds))
        cpu = {"value": rate, "unit": "mutants/s", "cores": threads, "kind": kind,
               "sample": f"the 16,384 seeds split over {threads} threads (havoc_mutant per slot, fresh Rng(1000+j)), {reps} passes in {dt:.1f} s"}
    ctx.close()
    return {"config": "BASELINE.json configs[3]: batched havoc mutation of 16,384 seeds (1-4 KB inputs), per-slot Rng, byte-exact vs ref",
            "value": n / (t["mean"] / 1e3), "unit": "mutants/s", "kernel_ms": t["mean"], "kernel_ms_min": t["min"], "iters": t["iters"],
            "mean_draws_per_mutant": float(want_draws.mean()),
            "roofline": roof(byts, t["mean"], peak, peak_src, "hfz_k_havoc",
                             "bytes = sum(in + out); the kernel is instruction-issue-bound, not HBM-bound"),
            "frac": byts / (t["mean"] / 1e3) / 1e9 / peak,
            "cpu_baseline": cpu,
            "parity_checked": "all 16,384 slots: mutant bytes, length, end Rng state, draw count",
            "l2_policy": "256 MB flush write before every timed launch (in + out = 100 MB would fit L2)"}


def bench_edge_and_large_map(hfz, dev, timer, peak, peak_src, args, threads):
    """configs[2]: synthetic basic-block traces (4 launches of 16 x 256 threads, ~205 k thread events
    per exec) -> edge record (K1); then 262,144-slot maps produced by K1 and folded by K2."""
    import torch
    from oracle import pyoracle
    n1 = args.edge_execs
    n2 = min(n1, args.large_execs)
    n_par = min(64, n2)
    t0 = time.time()
    tr = {k: np.ascontiguousarray(v) for k, v in synth().bb_traces(n1, seed=44).items()}
    gen_s = time.time() - t0
    d = traces_to_device(tr, dev)
    events = int(tr["sites"].size)
    n_threads = int(tr["thread_off"][-1])
    n_launch = int(tr["launch_off"][-1])

    def k1_bytes(n, H):
        nl = int(tr["launch_off"][n])
        nt = int(tr["thread_off"][nl])
        return 4 * int(tr["ev_off"][nt]) + 8 * (nt + nl) + 4 * H * n

    # ---- K1 alone, 65,536-slot maps
    ctx = hfz.Context(dev.index, S)
    raw = torch.zeros(n1 * REC, dtype=torch.uint8, device=dev)
    res = {}

    def run_k1():
        res["o"] = ctx.edge_record_batch(d["launch_off"], d["dims"], d["thread_off"], d["ev_off"], d["sites"], n1, raw=raw)

    run_k1()
    torch.cuda.synchronize()
    ck = pyoracle.best_checker(S)
    want_raw = np.zeros(n_par * REC, np.uint8)
    want_ev = np.zeros(n_par, np.uint64)
    ck.edge_record_range(tr, 0, n_par, S, want_raw, want_ev)
    if not (np.array_equal(raw[:n_par * REC].cpu().numpy(), want_raw)
            and np.array_equal(res["o"][1][:n_par].cpu().numpy().view(np.uint64), want_ev)):
        fail("K1 edge record (65,536-slot maps): device halves differ from the reference runtime")
    t_k1 = timer.run(run_k1, 10)
    cpu_k1 = None
    if not args.no_cpu:
        rate, kind, reps, dt, ns = cpu_edge_rate(tr, S, threads, 8, min(4.0, args.cpu_seconds))
        cpu_k1 = {"value": rate, "unit": "execs/s", "cores": threads, "kind": kind,
                  "sample": f"{ns} execs of the trace batch ({ns // threads} per thread) through hdvm::execute on a lambda-replay target, {reps} passes in {dt:.1f} s"}
    k1 = {"config": f"BASELINE.json configs[2] trace recipe, edge-record stage alone: {n1} execs, 4 launches x 16 blocks x 256 threads, "
                    f"{events / n1:.0f} thread events per exec, 65,536-slot maps",
          "value": n1 / (t_k1["mean"] / 1e3), "unit": "execs/s", "kernel_ms": t_k1["mean"], "kernel_ms_min": t_k1["min"],
          "iters": t_k1["iters"], "events_per_sec": events / (t_k1["mean"] / 1e3),
          "roofline": roof(k1_bytes(n1, S // 2), t_k1["mean"], peak, peak_src, "hfz_edge_record_batch: hfz_k_edge_classify + hfz_k_edge_divergent + hfz_k_edge_count (whole call)",
                           "bytes = 4 x events + 8 x (threads + launches) read + 4 x H written per exec; the time is the whole "
                           "C-ABI call (prep + scan launches, one D2H read of the queue sizes, then the three kernels); latency-bound"),
          "cpu_baseline": cpu_k1,
          "parity_checked": f"first {n_par} execs: device half of every record and warp_edge_events vs the reference runtime",
          "l2_policy": f"traces of {events * 4 / 1e6:.0f} MB + {n_threads * 8 / 1e6:.0f} MB of offsets per launch exceed L2",
          "trace_gen_seconds": round(gen_s, 1)}
    k1["frac"] = k1["roofline"]["frac"]
    del raw
    ctx.close()

    # ---- configs[2] proper: 262,144-slot maps from the traces, K1 -> K2
    c2 = hfz.Context(dev.index, S_LARGE)
    d2 = traces_to_device(trace_prefix(tr, n2), dev) if n2 != n1 else d
    raw2 = torch.zeros(n2 * REC_LARGE, dtype=torch.uint8, device=dev)

    def run_k1_large():
        res["l"] = c2.edge_record_batch(d2["launch_off"], d2["dims"], d2["thread_off"], d2["ev_off"], d2["sites"], n2, raw=raw2)

    run_k1_large()
    v2, cc2 = c2.new_virgin(), c2.new_edge_counts()
    # parity: n_par execs of the recipe through the 262,144-slot reference build, chained K1 -> K2
    o_par = c2.feedback_batch(raw2[:n_par * REC_LARGE], v2, cc2)
    torch.cuda.synchronize()
    ckl = pyoracle.best_checker(S_LARGE)
    want_raw = np.zeros(n_par * REC_LARGE, np.uint8)
    want_ev = np.zeros(n_par, np.uint64)
    ckl.edge_record_range(tr, 0, n_par, S_LARGE, want_raw, want_ev)
    vv, cc = np.zeros(S_LARGE, np.uint8), np.zeros(2, np.uint64)
    want = ckl.feedback_batch(want_raw, n_par, S_LARGE, vv, cc)
    ok = (np.array_equal(raw2[:n_par * REC_LARGE].cpu().numpy(), want_raw)
          and np.array_equal(res["l"][1][:n_par].cpu().numpy().view(np.uint64), want_ev)
          and np.array_equal(o_par["admit"].cpu().numpy(), want["admit"])
          and np.array_equal(o_par["sig_full"].cpu().numpy().view(np.uint64), want["sig_full"])
          and np.array_equal(o_par["sig_simple"].cpu().numpy().view(np.uint64), want["sig_simple"])
          and np.array_equal(o_par["nnz"].cpu().numpy().view(np.uint32), want["nnz"])
          and np.array_equal(v2.cpu().numpy(), vv) and np.array_equal(cc2.cpu().numpy().view(np.uint64), cc))
    if not ok:
        fail("configs[2] (262,144-slot maps from traces, K1 -> K2): GPU results differ from the reference")
    t_k1l = timer.run(run_k1_large, 10)
    # K2 on the maps K1 produced: warm = virgin after the first n2/4 maps; cold = empty virgin
    res["f"] = None

    def pre_cold():
        v2.zero_()
        cc2.zero_()

    def run_fold():
        res["f"] = c2.feedback_batch(raw2, v2, cc2, out=res["f"])

    t_k2 = timer.run(run_fold, 10, pre=pre_cold)
    admits = int((res["f"]["admit"] != 0).sum().item())
    cpu2 = None
    if not args.no_cpu:
        r1, kind1, reps1, dt1, ns = cpu_edge_rate(tr, S_LARGE, threads, 4, min(3.0, args.cpu_seconds))
        r2, kind2, reps2, dt2 = cpu_feedback_rate(want_raw, n_par, np.zeros(S_LARGE, np.uint8), threads,
                                                  min(3.0, args.cpu_seconds), slots=S_LARGE)
        cpu2 = {"value": 1.0 / (1.0 / r1 + 1.0 / r2), "unit": "execs/s", "cores": threads, "kind": kind1,
                "edge_record_execs_per_sec": r1, "fold_evals_per_sec": r2,
                "sample": f"edge record: {ns} execs ({ns // threads} per thread) through hdvm::execute, {reps1} passes in {dt1:.1f} s; "
                          f"fold: the {n_par} parity maps per replica from an empty virgin, {reps2} folds in {dt2:.1f} s (262,144-slot reference build)"}
    ms_chain = t_k1l["mean"] + t_k2["mean"]
    big = {"config": f"BASELINE.json configs[2]: 256 KB (262,144-slot) maps from synthetic basic-block traces incl. the edge-record stage: "
                     f"{n2} execs, K1 -> K2 chained on the device",
           "value": n2 / (ms_chain / 1e3), "unit": "execs/s", "ms_per_step": ms_chain, "iters": 10,
           "edge_record": {"value": n2 / (t_k1l["mean"] / 1e3), "unit": "execs/s", "kernel_ms": t_k1l["mean"], "kernel_ms_min": t_k1l["min"],
                           "counters": "per-exec shared-memory histogram in the count kernel, ranges of 32,768 slots per pass (no global atomic per hit)",
                           "roofline": roof(k1_bytes(n2, S_LARGE // 2), t_k1l["mean"], peak, peak_src, "hfz_edge_record_batch: classify + divergent + count (whole call)")},
           "fold": {"value": n2 / (t_k2["mean"] / 1e3), "unit": UNIT, "ms_per_step": t_k2["mean"], "ms_per_step_min": t_k2["min"],
                    "state": "empty virgin", "admits_per_step": admits,
                    "roofline": roof(n2 * REC_LARGE, t_k2["mean"], peak, peak_src, "whole step (scan + resolve + merge launches)")},
           "cpu_baseline": cpu2,
           "parity_checked": f"{n_par} execs of the recipe at S = 262,144 against the 262,144-slot reference build, chained: device halves + "
                             f"warp_edge_events from K1, then Admit codes, both signatures, nnz, final virgin and edge counters from K2 on those maps",
           "l2_policy": f"{n2 * REC_LARGE / 1e6:.0f} MB of maps and {events * 4 / 1e6 * n2 / n1:.0f} MB of traces per step exceed L2"}
    big["frac"] = big["fold"]["roofline"]["frac"]
    # ---- the same chain WITHOUT dense records in between: K1 writes per-exec touched-slot lists
    # (hfz_edge_record_batch_lists, raw_maps = NULL), K2 folds the lists (hfz_feedback_batch_sparse).
    # Checked against the dense chain above on every exec (which the reference pins on the first n_par).
    cap = 4096  # pairs per exec (the recipe touches ~2,100 distinct device slots per exec; an exec that did not fit would be reported)
    res["L"] = None

    def run_k1_lists():
        res["L"] = c2.edge_record_batch_lists(d2["launch_off"], d2["dims"], d2["thread_off"], d2["ev_off"], d2["sites"], n2,
                                              cap=cap, out=res["L"])

    run_k1_lists()
    res["g"] = None

    def run_fold_lists():
        res["g"] = c2.feedback_batch_sparse(res["L"]["entries"], res["L"]["entry_off"], v2, cc2, out=res["g"])

    pre_cold()
    run_fold()
    v_dense, c_dense = v2.clone(), cc2.clone()
    pre_cold()
    run_fold_lists()
    torch.cuda.synchronize()
    listed = int((res["L"]["n_slots"] >= 0).sum().item())
    same = (listed == n2 and torch.equal(res["L"]["events"], res["l"][1])
            and all(torch.equal(res["f"][k], res["g"][k]) for k in ("admit", "sig_full", "sig_simple", "nnz"))
            and torch.equal(v2, v_dense) and torch.equal(cc2, c_dense))
    if not same:
        fail("configs[2] list chain (K1 lists -> sparse fold) differs from the dense chain")
    t_k1s = timer.run(run_k1_lists, 10)
    t_k2s = timer.run(run_fold_lists, 10, pre=pre_cold)
    ms_lists = t_k1s["mean"] + t_k2s["mean"]
    big["lists_chain"] = {
        "what": "the same K1 -> K2 chain with per-exec touched-slot lists between the stages instead of dense 655,360-byte "
                "records: hfz_edge_record_batch_lists (raw_maps = NULL) -> hfz_feedback_batch_sparse",
        "value": n2 / (ms_lists / 1e3), "unit": "execs/s", "ms_per_step": ms_lists,
        "edge_record_ms": t_k1s["mean"], "fold_ms": t_k2s["mean"], "list_stride_pairs": cap,
        "mean_slots_per_exec": float(res["L"]["n_slots"].float().mean().item()),
        "parity_checked": f"all {n2} execs: warp_edge_events, Admit codes, both signatures, nnz, final virgin and edge counters equal the dense chain's"}
    c2.close()
    return k1, big


def scan_traffic(n):
    """roofline.traffic = DRAM bytes of one scan launch from the committed ncu capture -- attached only
    while the capture still describes the kernel that ran: the summary records the SHA-256 of the
    kernel source it profiled, and a capture of another source (or another batch size) is dropped."""
    for name in ("r2_scan_summary.json", "r1_scan_summary.json"):
        prof = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(prof):
            continue
        try:
            p = json.load(open(prof))
        except Exception:
            continue
        src = os.path.join(ROOT, "paper_2603_12485_b200", "csrc", "hfz_feedback.cu")
        sha = hashlib.sha256(open(src, "rb").read()).hexdigest()
        info = {"file": f"profiles/{name}", "kernel_source_sha256_at_capture": p.get("kernel_source_sha256"),
                "kernel_source_sha256_now": sha, "captured": p.get("captured")}
        if p.get("kernel_source_sha256") != sha:
            info["note"] = "capture is of an older kernel source: traffic withheld"
            return None, info
        if p.get("algorithmic_bytes_per_launch") != n * REC:
            info["note"] = "capture is of another batch size: traffic withheld"
            return None, info
        return p.get("dram_bytes_per_launch"), info
    return None, {"note": "no ncu capture committed"}


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_12485_b200 as hfz
    from paper_2603_12485_b200.sharding import ShardedFeedback

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback); use --impl reference for the CPU arm")
    # HFZ_BENCH_BACKEND=gloo maps every rank onto the visible GPUs round-robin (several ranks per
    # GPU): a functional check of the N > 1 path on a box with fewer GPUs -- never a bench number.
    backend = os.environ.get("HFZ_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    assert world == args.gpus or world == 1, f"WORLD_SIZE={world} but --gpus {args.gpus}"
    threads = os.cpu_count() or 1
    check = rank == 0 and not args.no_check

    n = args.execs
    ctx = hfz.Context(local_rank, S)
    ctx.set_option("time_scan", 1)
    # --- campaign state: virgin warmed by folding 4,096 maps (same on every rank)
    virgin = ctx.new_virgin()
    counts = ctx.new_edge_counts()
    warm_host = make_maps(4096, 1 << 24, args.mode)
    ctx.feedback_batch(torch.from_numpy(warm_host).to(dev), virgin, counts)
    v0 = virgin.clone()
    c0 = counts.clone()
    # --- the oracle folds the same maps as they are generated (rank 0): warm-up first
    ck = want = None
    if check:
        from oracle import pyoracle
        ck = pyoracle.best_checker(S)
        ov = np.zeros(S, np.uint8)
        oc = np.zeros(2, np.uint64)
        ck.feedback_batch(warm_host, 4096, S, ov, oc)
        if not (np.array_equal(v0.cpu().numpy(), ov) and np.array_equal(c0.cpu().numpy().view(np.uint64), oc)):
            fail("warm-up fold: virgin map / edge counters differ from the oracle")
        want = {"admit": np.zeros(n, np.uint8), "sig_full": np.zeros(n, np.uint64), "sig_simple": np.zeros(n, np.uint64)}
    # --- synthetic data: this rank's shard of the campaign batch, generated on the host in chunks
    t0 = time.time()
    raw = torch.empty(n * REC, dtype=torch.uint8, device=dev)
    chunk = 4096
    host_keep = None
    oracle_s = 0.0
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        a = make_maps(m, rank * n + i, args.mode)
        raw[i * REC:(i + m) * REC] = torch.from_numpy(a).to(dev)
        if i == 0:
            host_keep = a  # first chunk stays on the host: the cpu_baseline sample
        if check:
            t1 = time.time()
            w = ck.feedback_batch(a, m, S, ov, oc)  # sequential fold continues across chunks
            for k in want:
                want[k][i:i + m] = w[k]
            oracle_s += time.time() - t1
    gen_s = time.time() - t0 - oracle_s
    eng = ShardedFeedback(ctx, exchange=args.exchange)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    out = None

    def one_step():
        nonlocal out
        virgin.copy_(v0)  # every step folds the same batch into the same warmed state
        counts.copy_(c0)
        out = eng.step(raw, virgin, counts, out=out)

    for _ in range(max(3, args.warmup)):
        one_step()
    barrier()
    # --- parity against the oracle on EVERY exec of rank 0's shard (untimed): Admit codes in order, both
    # signatures; at N = 1 also the final virgin map and both edge counters
    parity = None
    if check:
        ok = (np.array_equal(out["sig_full"].cpu().numpy().view(np.uint64), want["sig_full"])
              and np.array_equal(out["sig_simple"].cpu().numpy().view(np.uint64), want["sig_simple"])
              and np.array_equal(out["admit"].cpu().numpy(), want["admit"]))
        if world == 1:
            ok = ok and np.array_equal(virgin.cpu().numpy(), ov) and np.array_equal(counts.cpu().numpy().view(np.uint64), oc)
        if not ok:
            fail("GPU results differ from the oracle")
        parity = {"checked": True, "execs": n, "checker": ck.kind, "oracle_seconds": round(oracle_s, 1),
                  "what": "every exec of rank 0's shard: Admit codes in order, Full and Simple signatures"
                          + ("; final virgin map; host/device edge counters" if world == 1 else
                             " (final virgin spans all ranks: compared in tests/test_sharding_gloo.py and the N = 1 run)")}

    ctx.get_stat("scan_ms_total")  # reset kernel-time accumulators
    launches0 = ctx.launch_count
    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.25)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        one_step()
    e1.record()
    barrier()
    ms_total = e0.elapsed_time(e1)
    scan_launches = args.steps
    scan_ms = ctx.get_stat("scan_ms_total")
    launches = ctx.launch_count - launches0
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    # nvidia-smi samples every 100 ms: keep the same load running a little longer.  A step holds a
    # collective when world > 1, so EVERY rank runs the same number of extra steps (derived from
    # the all-reduced time), not just the rank that samples.
    extra = 0
    if ms_total < 600:
        extra = int(700.0 / max(ms_total / args.steps, 1e-3)) + 1
        for _ in range(extra):
            one_step()
        torch.cuda.synchronize()
        ctx.get_stat("scan_ms_total")
    clocks = None
    if sampler:
        clocks = sampler.stop()
        if clocks is not None:
            clocks["note"] = (f"sampled over the timed region plus {extra} identical untimed steps"
                              if extra else "sampled over the timed region")
    ms_per_step = ms_total / args.steps
    value = world * n / (ms_per_step / 1e3)
    admits = int((out["admit"] != 0).sum().item())

    # --- stress mode (SURVEY 8d mode (i), N = 1 only): iid maps keep ~24 % of the batch admitted per
    # step even after the warm-up; the same device-resident step, 20 timed steps
    stress = None
    if world == 1 and args.mode == "campaign" and not args.no_stress:
        raw_s = torch.empty(n * REC, dtype=torch.uint8, device=dev)
        for i in range(0, n, chunk):
            m = min(chunk, n - i)
            raw_s[i * REC:(i + m) * REC] = torch.from_numpy(make_maps(m, i, "iid")).to(dev)
        vs, cs = ctx.new_virgin(), ctx.new_edge_counts()
        ctx.feedback_batch(torch.from_numpy(make_maps(4096, 1 << 24, "iid")).to(dev), vs, cs)
        vs0, cs0 = vs.clone(), cs.clone()
        out_s = None
        for _ in range(3):
            vs.copy_(vs0); cs.copy_(cs0)
            out_s = ctx.feedback_batch(raw_s, vs, cs, out=out_s)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(20):
            vs.copy_(vs0); cs.copy_(cs0)
            out_s = ctx.feedback_batch(raw_s, vs, cs, out=out_s)
        s1.record()
        torch.cuda.synchronize()
        ms_s = s0.elapsed_time(s1) / 20
        stress = {"mode": "iid", "value": n / (ms_s / 1e3), "unit": UNIT, "ms_per_step": ms_s, "steps": 20,
                  "admits_per_step": int((out_s["admit"] != 0).sum().item()),
                  "hbm_gbs_algorithmic": n * REC / (ms_s / 1e3) / 1e9}
        del raw_s, out_s
        ctx.get_stat("scan_ms_total")

    # --- end-to-end through the C-ABI with HOST buffers (pinned), copies inside the timed region.
    # Host forms of the same batch: (a) touched-slot lists -- what hetfuzz::b200::PackedBatch / CompactBatch /
    # SparseBatch keep per CoverageMap -- packed at 3 / 4 bytes per slot (hfz_feedback_batch_packed_host: the `e2e`
    # key), at 4 bytes per pair + wide pairs (hfz_feedback_batch_compact_host) and at 8 bytes per pair
    # (hfz_feedback_batch_sparse_host); (b) dense 163,840-byte records through
    # hfz_feedback_batch_host (PCIe-bound).
    e2e = None
    e2e_compact = None
    e2e_pairs = None
    e2e_dense = None
    if not args.no_e2e:
        n_e2e = args.e2e_execs or n
        v0_host = v0.cpu().numpy()
        c0_host = c0.cpu().numpy().view(np.uint64)

        def timed(call, steps):
            ts, res = [], None
            for i in range(1 + steps):
                vh, ch = v0_host.copy(), c0_host.copy()
                barrier()
                t1 = time.perf_counter()
                res = call(vh, ch)
                dt = time.perf_counter() - t1
                if i:
                    ts.append(dt)
            te = torch.tensor([float(np.mean(ts)), float(np.median(ts)), float(np.max(ts))], dtype=torch.float64, device=dev)
            tmin = torch.tensor([float(np.min(ts))], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
                dist.all_reduce(tmin, op=dist.ReduceOp.MAX)
            mean, med, mx = (float(x) for x in te.tolist())
            stats = {"steps": steps, "seconds_mean": mean, "seconds_median": med, "seconds_min": float(tmin.item()), "seconds_max": mx}
            return mean, stats, res

        # (a) touched-slot lists, built outside the timed region from the same maps
        ent_t, off_t = sparse_lists_from_device(raw, n_e2e, dev)
        ent_np, off_np = ent_t.numpy().view(np.uint32), off_t.numpy().view(np.uint64)

        def same_as_device_fold(res):
            return bool(np.array_equal(res["admit"], out["admit"][:n_e2e].cpu().numpy())
                        and np.array_equal(res["sig_full"], out["sig_full"][:n_e2e].cpu().numpy().view(np.uint64))
                        and np.array_equal(res["sig_simple"], out["sig_simple"][:n_e2e].cpu().numpy().view(np.uint64)))

        # (a1) 4 bytes per pair: compact words + wide pairs for counts >= 65,536
        comp_t, coff_t, wide_t, woff_t = compact_lists(ent_t, off_t)
        comp_np, coff_np = comp_t.numpy().view(np.uint32), coff_t.numpy().view(np.uint64)
        wide_np, woff_np = wide_t.numpy().view(np.uint32), woff_t.numpy().view(np.uint64)
        sec, stats, res = timed(lambda vh, ch: ctx.feedback_batch_compact_host(comp_np, coff_np, wide_np, woff_np, vh, ch),
                                args.e2e_steps)
        same = same_as_device_fold(res)
        if not same:
            fail("compact-list e2e results differ from the device-resident dense fold")
        e2e_compact = {"value": world * n_e2e / sec, "unit": UNIT,
               "h2d_bytes_per_step": int(comp_np.nbytes + coff_np.nbytes + wide_np.nbytes + woff_np.nbytes + S + 16),
               "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16 + 8),
               "execs_per_step": n_e2e, "timing": stats, "value_best": world * n_e2e / stats["seconds_min"],
               "value_median": world * n_e2e / stats["seconds_median"],
               "host_form": "touched-slot lists, 4 bytes per pair: u32 slot | count << 16 (counts < 65,536) + "
                            "(u32 slot, u32 count) pairs for larger device counters; random order inside an exec; "
                            "pinned host memory",
               "pairs_per_exec": float(ent_np.shape[0]) / n_e2e,
               "wide_pairs_per_exec": float(wide_np.shape[0]) / n_e2e,
               "equals_device_fold": same,
               "api": "hfz_feedback_batch_compact_host (lists streamed H2D chunk by chunk, ranked and folded on "
                      "the device)"}
        # (a3) the headline host form: packed lists -- 3 bytes per host-half slot, 4 per device-half slot
        h3_t, hoff_t, d17_t, doff_t = packed_lists(ent_t, off_t)
        h3_np, hoff_np = h3_t.numpy(), hoff_t.numpy().view(np.uint64)
        d17_np, doff_np = d17_t.numpy().view(np.uint32), doff_t.numpy().view(np.uint64)
        sec, stats, res = timed(lambda vh, ch: ctx.feedback_batch_packed_host(h3_np, hoff_np, d17_np, doff_np, vh, ch),
                                args.e2e_steps)
        same = same_as_device_fold(res)
        if not same:
            fail("packed-list e2e results differ from the device-resident dense fold")
        e2e = {"value": world * n_e2e / sec, "unit": UNIT,
               "h2d_bytes_per_step": int(h3_np.nbytes + hoff_np.nbytes + d17_np.nbytes + doff_np.nbytes + S + 16),
               "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16),
               "execs_per_step": n_e2e, "timing": stats, "value_best": world * n_e2e / stats["seconds_min"],
               "value_median": world * n_e2e / stats["seconds_median"],
               "host_form": "touched-slot lists, packed: host half 3 bytes per slot (slot lo, slot hi, count u8; every exec "
                            "padded to a multiple of four entries), device half 4 bytes per slot ((slot - 32768) | "
                            "min(count, 65536) << 15: the clip keeps every class of the device ladder); random order "
                            "inside an exec; pinned host memory",
               "pairs_per_exec": float(ent_np.shape[0]) / n_e2e,
               "equals_device_fold": same,
               "api": "hfz_feedback_batch_packed_host (lists streamed H2D chunk by chunk, ranked and folded on the device)"}
        del h3_t, hoff_t, d17_t, doff_t, h3_np, hoff_np, d17_np, doff_np
        # (a0) how fast the DEVICE side of that call is: the same lists already resident in HBM (8-byte pairs)
        # through hfz_feedback_batch_sparse -- rank + chain + resolve kernels, no PCIe
        lists_dev = None
        if world == 1:
            ent_d = ent_t.to(dev).view(torch.int32).reshape(-1, 2)
            off_d = off_t.to(dev).view(torch.int64)
            vd, cd, od = v0.clone(), c0.clone(), None
            for _ in range(2):
                vd.copy_(v0); cd.copy_(c0)
                od = ctx.feedback_batch_sparse(ent_d, off_d, vd, cd, out=od)
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            d0.record()
            for _ in range(10):
                vd.copy_(v0); cd.copy_(c0)
                od = ctx.feedback_batch_sparse(ent_d, off_d, vd, cd, out=od)
            d1.record()
            torch.cuda.synchronize()
            ms_d = d0.elapsed_time(d1) / 10
            if not (torch.equal(od["admit"], out["admit"][:n_e2e]) and torch.equal(od["sig_full"], out["sig_full"][:n_e2e])):
                fail("device-resident list fold differs from the dense fold")
            lists_dev = {"value": n_e2e / (ms_d / 1e3), "unit": UNIT, "ms_per_step": ms_d, "steps": 10,
                         "bytes_per_step": int(ent_d.numel() * 4),
                         "what": "the same touched-slot lists already in HBM (8 bytes per pair) through "
                                 "hfz_feedback_batch_sparse: what the host calls above would run at without PCIe"}
            del ent_d, off_d, vd, cd, od
            e2e["lists_device_resident"] = lists_dev
        # (a2) the same lists at 8 bytes per pair
        sec, stats, res = timed(lambda vh, ch: ctx.feedback_batch_sparse_host(ent_np, off_np, vh, ch), args.e2e_steps)
        if not same_as_device_fold(res):
            fail("sparse e2e results differ from the device-resident dense fold")
        e2e_pairs = {"value": world * n_e2e / sec, "unit": UNIT,
                     "h2d_bytes_per_step": int(ent_np.nbytes + off_np.nbytes + S + 16),
                     "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16 + 8), "execs_per_step": n_e2e,
                     "timing": stats,
                     "host_form": "touched-slot lists, 8 bytes per pair: (u32 slot, u32 count)",
                     "api": "hfz_feedback_batch_sparse_host"}
        del ent_t, off_t, ent_np, off_np, comp_t, coff_t, wide_t, woff_t, comp_np, coff_np, wide_np, woff_np
        # (b) dense records
        # the dense form pins 10.7 GB of host memory per rank: single-rank runs only
        if not args.no_e2e_dense and world == 1:
            pinned = torch.empty(n_e2e * REC, dtype=torch.uint8, pin_memory=True)
            pinned.copy_(raw[: n_e2e * REC])
            raw_host = pinned.numpy()
            sec, stats, res = timed(lambda vh, ch: ctx.feedback_batch_host(raw_host, vh, ch), min(3, args.e2e_steps))
            e2e_dense = {"value": world * n_e2e / sec, "unit": UNIT,
                         "h2d_bytes_per_step": int(n_e2e * REC + S + 16),
                         "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16),
                         "execs_per_step": n_e2e, "timing": stats, "host_form": "dense 163,840-byte records, pinned host memory",
                         "api": "hfz_feedback_batch_host (chunked overlapped H2D); PCIe-bound"}
            del pinned

    # --- the CoverageMap-to-results harness (C++: the reference's own types on the host side)
    e2e_cm = None
    if rank == 0 and world == 1 and not args.no_e2e and not args.no_harness:
        e2e_cm = run_coveragemap_harness(args)

    peak, peak_src = hbm_peak()
    extra_cfg = {}
    if world == 1 and not args.no_configs:
        timer = GpuTimer(dev)
        extra_cfg["config0_small_batch"] = bench_config0(hfz, dev, timer, peak, peak_src, args, threads)
        extra_cfg["k3_havoc"] = bench_havoc(hfz, dev, timer, peak, peak_src, args, threads)
        k1, big = bench_edge_and_large_map(hfz, dev, timer, peak, peak_src, args, threads)
        extra_cfg["k1_edge_record"] = k1
        extra_cfg["config2_large_map"] = big

    if rank == 0:
        algo_bytes = n * REC  # 163,840 B read per eval x evals per launch
        achieved = algo_bytes / (scan_ms / scan_launches / 1e3) / 1e9
        traffic, traffic_src = scan_traffic(n)
        roofline = {"bound": "hbm", "kernel": "hfz_k_scan", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": algo_bytes,
                    "kernel_ms_per_launch": scan_ms / scan_launches,
                    "step_frac": (world * n * REC / (ms_per_step / 1e3) / 1e9) / (peak * world)}
        cpu = None
        if world == 1 and not args.no_cpu:
            rate, kind, reps, dt = cpu_feedback_rate(host_keep[: args.cpu_sample * REC], args.cpu_sample,
                                                     v0.cpu().numpy(), threads, args.cpu_seconds)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": f"first {args.cpu_sample} maps of the batch per replica, {threads} independent "
                             f"replicas with private pre-warmed virgin maps, {reps} replica folds in {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32->u64", "data": "synthetic",
            "config": base_config(args, world),
            "run_info": {"admits_per_step_rank0": admits, "gen_seconds": round(gen_s, 1)},
            "parity": parity, "parity_checked": bool(parity and parity["checked"]),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_compact": e2e_compact, "e2e_pairs": e2e_pairs, "e2e_dense": e2e_dense,
            "e2e_from_coveragemap": e2e_cm,
            "stress_mode": stress,
            "gpu_launches": launches,
            "clocks": clocks,
            "hbm_gbs_algorithmic": world * n * REC / (ms_per_step / 1e3) / 1e9,
            "logical_map_gbs": world * n * S / (ms_per_step / 1e3) / 1e9,
        }
        line.update(extra_cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        eng.close()  # peers exchange: unmap / free the shared delta buffers (barrier inside)
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def run_coveragemap_harness(args):
    """bench/e2e_coveragemap (C++): builds hetfuzz::CoverageMap objects from the synthetic recipe, then
    times PackedBatch::append x N + the fold + result read-back as one region, and the reference's
    engine.cpp:471-478 loop on the same maps in the same binary.  Returns its JSON or a reason."""
    exe = os.path.join(ROOT, "bench", "e2e_coveragemap")
    if not os.path.exists(exe):
        return {"unavailable": "bench/e2e_coveragemap not built (run __graft_entry__.build())"}
    try:
        r = subprocess.run([exe, "--execs", str(args.harness_execs), "--steps", str(args.harness_steps)],
                           capture_output=True, text=True, timeout=900, cwd=ROOT)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"harness failed to run: {e}"}
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        return {"unavailable": f"harness rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"}
    return json.loads(lines[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--execs", type=int, default=65536, help="executions per GPU per step")
    ap.add_argument("--mode", default="campaign", choices=["campaign", "iid"])
    ap.add_argument("--cpu-sample", type=int, default=2048)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-execs", type=int, default=0)
    ap.add_argument("--edge-execs", type=int, default=2048, help="execs of the configs[2] trace batch (K1)")
    ap.add_argument("--large-execs", type=int, default=1024, help="execs of the 262,144-slot K1 -> K2 chain")
    ap.add_argument("--harness-execs", type=int, default=65536)
    ap.add_argument("--harness-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-dense", action="store_true")
    ap.add_argument("--no-harness", action="store_true")
    ap.add_argument("--no-stress", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[0]/[2]/[3] sub-benchmarks")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "peers"],
                    help="N > 1: NCCL allgather of the deltas (default) or peer-memory loads from CUDA IPC "
                         "buffers (hfz_peer_alloc / hfz_peer_open + hfz_feedback_resolve_peers)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
