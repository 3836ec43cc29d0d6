#!/usr/bin/env python
"""Headline benchmark: coverage-map evals/sec of the fused feedback step (BASELINE.json).

    python bench.py --gpus N --steps K --warmup W [--impl reference]

A "step" is one pass of the hot path (classify + has_new_bits + 2 signatures + virgin fold)
over one batch of synthetic raw maps: configs[1] of BASELINE.json, a 65,536-exec batch of
64 KB (65,536-slot) maps per GPU, ~2 % density, campaign-like novelty, virgin pre-warmed with
4,096 maps.  N > 1 (launched by torchrun, one rank per GPU) shards the campaign batch
(N x 65,536 execs), allgathers the per-rank novelty deltas over NCCL and merges in rank order
("scaling": "weak").  Prints ONE JSON line on rank 0.
"""
import argparse
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
METRIC = "coverage_map_evals_per_sec"
UNIT = "evals/s"


def make_maps(n, first, mode):
    from paper_2603_12485_b200 import synth
    gen = synth.maps_campaign if mode == "campaign" else synth.maps_iid
    return gen(n, S, first=first)


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


# --------------------------------------------------------------------------- CPU baseline
def cpu_feedback_rate(raw_sample, n_sample, v0, threads, min_seconds, reps_cap=64):
    """Reference CPU path (classify_trace + 2x trace_signature + has_new_bits, engine.cpp:471-478)
    on `threads` host threads, each folding the whole sample as an independent replica with a
    private pre-warmed virgin map.  Returns (evals/s, kind, reps, seconds)."""
    from oracle import pyoracle
    if pyoracle.Ref.available(S):
        ck = pyoracle.Ref(S)
        h = ck.maps_create(raw_sample, n_sample)  # CoverageMap objects, outside the timed region

        def fold(v, c):
            ck.feedback_run(h, 0, n_sample, v, c)
    else:
        ck = pyoracle.Port()
        h = None
        adm = [np.zeros(n_sample, np.uint8) for _ in range(threads)]
        sf = [np.zeros(n_sample, np.uint64) for _ in range(threads)]
        ss = [np.zeros(n_sample, np.uint64) for _ in range(threads)]
        nz = [np.zeros(n_sample, np.uint32) for _ in range(threads)]
        tl = threading.local()

        def fold(v, c, _i=[0]):
            i = getattr(tl, "i", None)
            if i is None:
                i = tl.i = _i[0]
                _i[0] += 1
            ck._feedback(raw_sample, n_sample, S, v, c, None, adm[i], sf[i], ss[i], nz[i])

    done = [0] * threads
    stop_at = [None]

    def worker(i):
        reps = 0
        while True:
            v = v0.copy()
            c = np.zeros(2, np.uint64)
            fold(v, c)
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
    if h is not None:
        ck.maps_free(h)
    total = sum(done) * n_sample
    return total / dt, ck.kind, sum(done), dt


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sample = args.cpu_sample
    raw = make_maps(n_sample, 0, args.mode)
    warm = make_maps(4096, 1 << 24, args.mode)
    from oracle import pyoracle
    port = pyoracle.Port()
    v0 = np.zeros(S, np.uint8)
    port.feedback_batch(warm, 4096, S, v0, np.zeros(2, np.uint64))
    for _ in range(args.warmup):
        cpu_feedback_rate(raw, n_sample, v0, threads, 0.0, reps_cap=1)
    rates, secs = [], 0.0
    kind = "port"
    for _ in range(args.steps):
        r, kind, reps, dt = cpu_feedback_rate(raw, n_sample, v0, threads, args.cpu_seconds / max(1, args.steps))
        rates.append(r)
        secs += dt
    value = float(np.mean(rates))
    sample = (f"{n_sample} maps of the workload per replica, {threads} independent replicas "
              f"(private pre-warmed virgin), each step ~{args.cpu_seconds / max(1, args.steps):.1f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / max(1, args.steps) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32->u64", "data": "synthetic",
        "config": {"workload": workload_name(args), "map_slots": S, "bytes_per_eval": REC,
                   "execs_per_gpu": args.execs, "density": 0.02, "mode": args.mode},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_name(args):
    return (f"BASELINE.json configs[1]: {args.execs}-exec batch of 64 KB (65,536-slot) maps per GPU, "
            f"fused classify+has_new_bits+signatures, {args.mode}-like novelty, virgin pre-warmed with 4,096 maps")


# --------------------------------------------------------------------------- GPU arm
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

    n = args.execs
    ctx = hfz.Context(local_rank, S)
    ctx.set_option("time_scan", 1)
    # --- synthetic data: this rank's shard of the campaign batch, generated on the host in chunks
    t0 = time.time()
    raw = torch.empty(n * REC, dtype=torch.uint8, device=dev)
    chunk = 4096
    host_keep = None
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        a = make_maps(m, rank * n + i, args.mode)
        raw[i * REC:(i + m) * REC] = torch.from_numpy(a).to(dev)
        if i == 0:
            host_keep = a  # first chunk stays on the host: parity check + cpu_baseline sample
    gen_s = time.time() - t0
    # --- campaign state: virgin warmed by folding 4,096 maps (same on every rank)
    virgin = ctx.new_virgin()
    counts = ctx.new_edge_counts()
    warm_host = make_maps(4096, 1 << 24, args.mode)
    ctx.feedback_batch(torch.from_numpy(warm_host).to(dev), virgin, counts)
    v0 = virgin.clone()
    c0 = counts.clone()
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
    # --- parity spot check against the oracle on the first 512 execs of rank 0's shard (untimed)
    parity = None
    if rank == 0 and not args.no_check:
        from oracle import pyoracle
        ck = pyoracle.best_checker(S)
        vv = v0.cpu().numpy().copy()
        cc = c0.cpu().numpy().view(np.uint64).copy()
        want = ck.feedback_batch(host_keep[:512 * REC], 512, S, vv, cc)
        got_f = out["sig_full"][:512].cpu().numpy().view(np.uint64)
        got_s = out["sig_simple"][:512].cpu().numpy().view(np.uint64)
        got_a = out["admit"][:512].cpu().numpy()
        parity = bool(np.array_equal(got_f, want["sig_full"]) and np.array_equal(got_s, want["sig_simple"])
                      and np.array_equal(got_a, want["admit"]))
        if not parity:
            raise SystemExit("bench.py: GPU results differ from the oracle -- refusing to report a number")

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
    # Host forms of the same batch: (a) touched-slot lists -- what hetfuzz::b200::CompactBatch /
    # SparseBatch keep per CoverageMap -- at 4 bytes per pair (hfz_feedback_batch_compact_host) and at
    # 8 bytes per pair (hfz_feedback_batch_sparse_host); (b) dense 163,840-byte records through
    # hfz_feedback_batch_host (PCIe-bound).
    e2e = None
    e2e_pairs = None
    e2e_dense = None
    if not args.no_e2e:
        n_e2e = args.e2e_execs or n
        v0_host = v0.cpu().numpy()
        c0_host = c0.cpu().numpy().view(np.uint64)

        def timed(call):
            ts, res = [], None
            for i in range(1 + args.e2e_steps):
                vh, ch = v0_host.copy(), c0_host.copy()
                barrier()
                t1 = time.perf_counter()
                res = call(vh, ch)
                dt = time.perf_counter() - t1
                if i:
                    ts.append(dt)
            te = torch.tensor([float(np.mean(ts))], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return float(te.item()), res

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
        sec, res = timed(lambda vh, ch: ctx.feedback_batch_compact_host(comp_np, coff_np, wide_np, woff_np, vh, ch))
        same = same_as_device_fold(res)
        if not same:
            raise SystemExit("bench.py: compact-list e2e results differ from the device-resident dense fold")
        e2e = {"value": world * n_e2e / sec, "unit": UNIT,
               "h2d_bytes_per_step": int(comp_np.nbytes + coff_np.nbytes + wide_np.nbytes + woff_np.nbytes + S + 16),
               "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16 + 8),
               "execs_per_step": n_e2e,
               "host_form": "touched-slot lists, 4 bytes per pair: u32 slot | count << 16 (counts < 65,536) + "
                            "(u32 slot, u32 count) pairs for larger device counters; random order inside an exec; "
                            "pinned host memory",
               "pairs_per_exec": float(ent_np.shape[0]) / n_e2e,
               "wide_pairs_per_exec": float(wide_np.shape[0]) / n_e2e,
               "equals_device_fold": same,
               "api": "hfz_feedback_batch_compact_host (lists streamed H2D chunk by chunk, ranked and folded on "
                      "the device)"}
        # (a2) the same lists at 8 bytes per pair
        sec, res = timed(lambda vh, ch: ctx.feedback_batch_sparse_host(ent_np, off_np, vh, ch))
        if not same_as_device_fold(res):
            raise SystemExit("bench.py: sparse e2e results differ from the device-resident dense fold")
        e2e_pairs = {"value": world * n_e2e / sec, "unit": UNIT,
                     "h2d_bytes_per_step": int(ent_np.nbytes + off_np.nbytes + S + 16),
                     "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16 + 8), "execs_per_step": n_e2e,
                     "host_form": "touched-slot lists, 8 bytes per pair: (u32 slot, u32 count)",
                     "api": "hfz_feedback_batch_sparse_host"}
        del ent_t, off_t, ent_np, off_np, comp_t, coff_t, wide_t, woff_t, comp_np, coff_np, wide_np, woff_np
        # (b) dense records
        # the dense form pins 10.7 GB of host memory per rank: single-rank runs only
        if not args.no_e2e_dense and world == 1:
            pinned = torch.empty(n_e2e * REC, dtype=torch.uint8, pin_memory=True)
            pinned.copy_(raw[: n_e2e * REC])
            raw_host = pinned.numpy()
            sec, res = timed(lambda vh, ch: ctx.feedback_batch_host(raw_host, vh, ch))
            e2e_dense = {"value": world * n_e2e / sec, "unit": UNIT,
                         "h2d_bytes_per_step": int(n_e2e * REC + S + 16),
                         "d2h_bytes_per_step": int(n_e2e * (1 + 8 + 8 + 4) + S + 16),
                         "execs_per_step": n_e2e, "host_form": "dense 163,840-byte records, pinned host memory",
                         "api": "hfz_feedback_batch_host (chunked overlapped H2D); PCIe-bound"}
            del pinned

    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(peaks_path):
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        algo_bytes = n * REC  # 163,840 B read per eval x evals per launch
        achieved = algo_bytes / (scan_ms / scan_launches / 1e3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "r1_scan_summary.json")
        if os.path.exists(prof) and n == 65536:  # the ncu capture is of the default workload
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "kernel": "hfz_k_scan", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": algo_bytes,
                    "kernel_ms_per_launch": scan_ms / scan_launches,
                    "step_frac": (world * n * REC / (ms_per_step / 1e3) / 1e9) / (peak * world)}
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            rate, kind, reps, dt = cpu_feedback_rate(host_keep[: args.cpu_sample * REC], args.cpu_sample,
                                                     v0.cpu().numpy(), threads, args.cpu_seconds)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": f"first {args.cpu_sample} maps of the batch per replica, {threads} independent "
                             f"replicas with private pre-warmed virgin maps, {reps} replica folds in {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8/u32->u64", "data": "synthetic",
            "config": {"workload": workload_name(args), "map_slots": S, "bytes_per_eval": REC,
                       "execs_per_gpu": n, "global_execs_per_step": world * n, "density": 0.02, "mode": args.mode,
                       "l2_policy": (f"inputs larger than L2 ({n * REC / 1e9:.1f} GB per GPU per step)" if n * REC > 512e6
                                     else f"inputs of {n * REC / 1e6:.0f} MB per GPU may stay L2-resident (not a bench configuration)"),
                       "admits_per_step_rank0": admits, "parallelism": f"exec-sharded x{world}",
                       "gen_seconds": round(gen_s, 1), "parity_checked": parity},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_pairs": e2e_pairs, "e2e_dense": e2e_dense,
            "stress_mode": stress,
            "gpu_launches": launches,
            "clocks": clocks,
            "hbm_gbs_algorithmic": world * n * REC / (ms_per_step / 1e3) / 1e9,
            "logical_map_gbs": world * n * S / (ms_per_step / 1e3) / 1e9,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-execs", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-e2e-dense", action="store_true")
    ap.add_argument("--no-stress", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "peers"],
                    help="N > 1: NCCL allgather of the deltas (default) or peer-memory loads through torch "
                         "symmetric memory (hfz_feedback_resolve_peers)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
