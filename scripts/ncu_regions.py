"""Summarise an ncu report of the scan kernel: headline metrics + instruction counts per code region."""
import csv, subprocess, sys
rep = sys.argv[1]
grouprows = float(sys.argv[2]) if len(sys.argv) > 2 else 1332 * 2 * 320
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__inst_executed.avg.per_cycle_elapsed', 'launch__registers_per_thread',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'launch__block_size', 'launch__grid_size', 'smsp__average_warp_latency_per_inst_issued.ratio',
        'smsp__warps_eligible.avg.per_cycle_active', 'lts__t_sector_hit_rate.pct', 'smsp__cycles_elapsed.avg.per_second',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed']
for i, h in enumerate(hdr):
    if h in want or ('issue_stalled' in h and h.endswith('_per_warp_active.pct')):
        print(f"{h:88s} {vals[i]:>18s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
isrc, iex, ismp, iavg = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('# Samples'), hdr.index('Avg. Threads Executed')
data = []
for r in rows[2:]:
    try:
        data.append((r[isrc], int(r[iex]), int(r[ismp]), float(r[iavg])))
    except Exception:
        pass
tot = sum(d[1] for d in data); tots = sum(d[2] for d in data)
print("total inst", tot, "per grouprow", tot / grouprows)
B = 40
for s in range(0, len(data), B):
    blk = data[s:s + B]
    ex = sum(d[1] for d in blk); sm = sum(d[2] for d in blk)
    if ex > tot * 0.005 or sm > tots * 0.005:
        ops = {}
        for d in blk:
            t = d[0].split()
            o = t[1] if t[0].startswith('@') else t[0]
            ops[o.split('.')[0]] = ops.get(o.split('.')[0], 0) + d[1]
        top = sorted(ops.items(), key=lambda x: -x[1])[:6]
        thr = sum(d[3] * d[1] for d in blk) / max(ex, 1)
        print(f"{s:5d}-{s+B:5d} ex={ex/tot*100:5.1f}% ({ex/grouprows:7.1f}/grouprow) smp={sm/tots*100:5.1f}% thr={thr:4.1f} "
              + " ".join(f"{k}:{v/grouprows:.0f}" for k, v in top))
