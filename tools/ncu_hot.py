"""Summarise an ncu report: stall reasons and the hottest SASS lines.
usage: python tools/ncu_hot.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, vals = r[0], r[2]
print("== stalls (per issued instruction)")
for h, v in zip(hdr, vals):
    if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
        try:
            f = float(v.replace(",", ""))
        except ValueError:
            continue
        if f > 0.03:
            print(f"  {h.split('stalled_')[1].split('_per_issue')[0]:24s} {f:.3f}")
for h, v in zip(hdr, vals):
    if h in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"):
        print(" ", h, v)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
lines = []
ops = collections.Counter()
for row in rows[2:]:
    try:
        s = float(row[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = float(row[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    text = row[ix["Source"]].strip()
    lines.append((s, n, row[ix["Address"]][-5:], text))
    tok = text.split()
    if tok:
        op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
        ops[op.split(".")[0]] += n
tot = sum(x[0] for x in lines)
print(f"== instruction mix (warp-level executed): {ops.most_common(14)}")
print(f"== top {top} SASS lines by stall samples (total {tot:.0f})")
for s, n, a, t in sorted(lines, reverse=True)[:top]:
    print(f"  {s:8.0f} {100*s/tot:5.1f}%  n={n:10.0f}  {a}  {t[:90]}")
