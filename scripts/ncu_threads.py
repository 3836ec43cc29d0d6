"""Per CUDA source line: executed warp instructions and average active threads (divergence), from an
ncu report with source.  usage: ncu_threads.py report.ncu-rep lo-hi[,lo-hi...] [min_inst] [kernel regex]"""
import csv, subprocess, sys
rep = sys.argv[1]
ranges = [tuple(int(x) for x in r.split("-")) for r in sys.argv[2].split(",")]
min_inst = int(sys.argv[3]) if len(sys.argv) > 3 else 0
kf = ["-k", "regex:" + sys.argv[4]] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[hi]
iex, ith = h.index("Instructions Executed"), h.index("Avg. Threads Executed")
for r in rows[hi + 1:]:
    if len(r) <= ith or not r[0].strip():
        continue
    try:
        n, ex = int(r[0]), int(r[iex])
    except ValueError:
        continue
    if any(lo <= n <= hi_ for lo, hi_ in ranges) and ex >= min_inst:
        print(f"L{n:5d} inst {ex:>11d} thr {r[ith]:>3s}  {r[1].strip()[:100]}")
