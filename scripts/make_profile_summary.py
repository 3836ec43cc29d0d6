"""Turn gpurun_out/ ncu captures into the tracked summaries under profiles/ (named per round)."""
import collections, csv, json, os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
rep = os.path.join(ROOT, "gpurun_out", f"{rnd}_scan.ncu-rep")
launches = os.path.join(ROOT, "gpurun_out", f"{rnd}_bench_launches.csv")
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}
def num(k):
    return float(m[k][0].replace(",", ""))
def scaled(k):
    v, u = m[k]
    v = float(v.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}
    return v * mult.get(u, 1.0)
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "lts__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__cycles_elapsed.avg.per_second", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "launch__shared_mem_per_block_dynamic"]
sel = {k: {"value": m[k][0], "unit": m[k][1]} for k in keys if k in m}
stalls = {h: m[h][0] for h in hdr if "issue_stalled" in h and h.endswith("_per_warp_active.pct")}
dur = scaled("gpu__time_duration.sum")
rd, wr = scaled("dram__bytes_read.sum"), scaled("dram__bytes_write.sum")
import hashlib, time
summary = {
    "round": rnd, "kernel": m["Kernel Name"][0] if "Kernel Name" in m else "hfz_k_scan",
    # bench.py attaches roofline.traffic only while this hash still matches the kernel source it runs
    "kernel_source_sha256": hashlib.sha256(open(os.path.join(ROOT, "paper_2603_12485_b200", "csrc", "hfz_feedback.cu"), "rb").read()).hexdigest(),
    "captured": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime(os.path.getmtime(rep))),
    "command": "ncu --set full --clock-control none --import-source on -k regex:hfz_k_scan -s 4 -c 1 "
               "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu",
    "duration_s_under_ncu": dur, "dram_bytes_read": rd, "dram_bytes_write": wr,
    "dram_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": 65536 * 163840,
    "traffic_over_algorithmic": (rd + wr) / (65536 * 163840),
    "dram_gbs_under_ncu": (rd + wr) / dur / 1e9, "metrics": sel, "stall_pct_per_warp_active": stalls,
}
if "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum" in m and "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum" in m:
    summary["sectors_per_global_load_request"] = num("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") / num(
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
json.dump(summary, open(os.path.join(out, f"{rnd}_scan_summary.json"), "w"), indent=1)
if os.path.exists(launches):
    shutil.copy(launches, os.path.join(out, f"{rnd}_bench_launches.csv"))
    rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    h = rows[0]; ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ik].split("(")[0][-48:], []).append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for k, v in agg.items() if "hfz_k" in k)
    with open(os.path.join(out, f"{rnd}_bench_launches_summary.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e-dense --e2e-steps 1\n")
        f.write("# (timed steps, the untimed clock-sampling steps, torch data-prep kernels of the sparse lists, then the sparse e2e calls)\n")
        f.write("# per-launch times are cold-cache and serialised: compare SHARES\n")
        for k, v in agg.items():
            share = f"{sum(v)/tot*100:5.1f}% of hfz kernels" if "hfz_k" in k else ""
            f.write(f"{k:50s} n={len(v):3d} total_us={sum(v)/1e3:10.1f} mean_us={sum(v)/len(v)/1e3:9.1f} {share}\n")
reg = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_regions.py"), rep], capture_output=True, text=True).stdout
open(os.path.join(out, f"{rnd}_scan_regions.txt"), "w").write(reg)
print(json.dumps({k: summary[k] for k in ("duration_s_under_ncu", "dram_bytes_per_launch", "traffic_over_algorithmic", "dram_gbs_under_ncu", "sectors_per_global_load_request") if k in summary}))


# ---- secondary kernels: one compact summary per extra report found in gpurun_out/
EXTRA = {"scan_pipe": "scripts/probe_feedback.py --n 4096 --configs '' --reps 1 --sweep 4096 (-k regex:hfz_k_scan_pipe -s 2 -c 1)",
         "expand": "scripts/probe_sparse.py --execs 16384 --chunks 8192 (-k regex:hfz_k_expand -s 2 -c 2)",
         "edge": "EDGE_FLAT=0 scripts/probe_k1k3.py edge (-k regex:hfz_k_edge_record -c 1): the per-exec kernel (round 1's design; since round 2 only execs whose launches differ in geometry)",
         "edge_flat": "EDGE_N=1024 scripts/probe_k1k3.py edge (-k regex:hfz_k_edge_(classify|divergent|count) -s 3 -c 3): the flat path's three kernels on 1,024 execs of the configs[2] trace recipe",
         "edge_flat_large": "EDGE_N=1024 EDGE_S=262144 scripts/probe_k1k3.py edge (same three kernels, 262,144-slot map: the count kernel takes the device half in four ranges)",
         "small_step": "scripts/probe_small.py (-k regex:hfz_k_small_step -s 8 -c 1): the fused small-batch step",
         "havoc": "scripts/probe_k1k3.py havoc (-k regex:hfz_k_havoc -s 2 -c 1)",
         "sparse": "scripts/probe_sparse.py --chunks 65536 (-k regex:hfz_k_sparse -s 6 -c 2: rank + chain of one 65,536-exec device call)"}
for name, cmd in EXTRA.items():
    rp = os.path.join(ROOT, "gpurun_out", f"{rnd}_{name}.ncu-rep")
    if not os.path.exists(rp):
        continue
    raw2 = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows2 = list(csv.reader(raw2.splitlines()))
    hdr2, units2 = rows2[0], rows2[1]
    outl = []
    for vals2 in rows2[2:]:
        mm = {h: (vals2[i], units2[i]) for i, h in enumerate(hdr2)}
        sel2 = {k: {"value": mm[k][0], "unit": mm[k][1]} for k in keys if k in mm}
        st2 = {h: mm[h][0] for h in hdr2 if "issue_stalled" in h and h.endswith("_per_warp_active.pct")}
        top = dict(sorted(st2.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:6])
        outl.append({"kernel": mm.get("Kernel Name", ("?",))[0], "metrics": sel2, "top_stalls_pct_per_warp_active": top})
    json.dump({"round": rnd, "command": "ncu --set full --clock-control none python " + cmd, "launches": outl},
              open(os.path.join(out, f"{rnd}_{name}_summary.json"), "w"), indent=1)
