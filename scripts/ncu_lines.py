"""Per CUDA source line: executed warp instructions and stall samples, from an ncu report captured
with --import-source on (kernels compiled with -lineinfo).  usage: ncu_lines.py report.ncu-rep [top N]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + kfilter, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
iline, isrc = hdr.index("Line No"), hdr.index("Source")
iex, ism = hdr.index("Instructions Executed"), hdr.index("# Samples")
agg = collections.OrderedDict()
cur = None
tot_ex = tot_sm = 0
for r in rows[hi + 1:]:
    if len(r) <= max(iex, ism):
        continue
    if r[iline].strip():            # a CUDA source line header row
        cur = (r[iline].strip(), r[isrc].strip()[:110])
        agg.setdefault(cur, [0, 0])
        continue
    try:
        ex, sm = int(r[iex]), int(r[ism])
    except ValueError:
        continue
    if cur is None:
        continue
    agg[cur][0] += ex
    agg[cur][1] += sm
    tot_ex += ex
    tot_sm += sm
print(f"total warp instructions {tot_ex}, samples {tot_sm}")
for (ln, src), (ex, sm) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ex / max(tot_ex, 1) * 100:5.1f}% inst {sm / max(tot_sm, 1) * 100:5.1f}% stall  L{ln:>5s}  {src}")
