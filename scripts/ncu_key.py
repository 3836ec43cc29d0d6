"""Key metrics of every kernel in an ncu report (raw page).  usage: ncu_key.py report.ncu-rep [kernel regex]"""
import csv, subprocess, sys
rep = sys.argv[1]
kf = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_static", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "smsp__inst_executed_op_shared_atom.sum", "smsp__inst_executed_op_global_red.sum",
        "smsp__inst_executed_op_generic_atom_dot_alu.sum",
        "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
STALL = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:110])
    for k in KEYS:
        if k in h:
            print(f"  {k:70s} {r[h.index(k)]} {rows[1][h.index(k)]}")
    st = sorted(((float(r[h.index(c)] or 0), c) for c in STALL), reverse=True)[:7]
    print("  stalls/issue:", ", ".join(f"{c.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}" for v, c in st))
