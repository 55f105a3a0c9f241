"""Attribute an ncu source-page (SASS) capture to CUDA source lines.

  python tools/ncu_lines.py <report.ncu-rep> <cubin> <mangled-kernel-name> [top]

ncu's --page source --csv lists the kernel's SASS in address order with warp
stall samples per instruction; `nvdisasm -g` of the same cubin maps every
instruction offset to file:line (the innermost inlined line).  Prints the
stall-sample share and executed instructions per source line."""
import csv
import collections
import re
import subprocess
import sys

rep, cubin, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr = rows[1]
data = rows[2:]
iss = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
on, cur, lines = False, None, {}
for ln in sass.splitlines():
    if ".section" in ln:
        on = (".text." + fun) in ln
        continue
    if not on:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m:
        lines[int(m.group(1), 16) // 16] = cur
assert len(lines) == len(data), (len(lines), len(data))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
tot = 0.0
for i, r in enumerate(data):
    s = float(r[iss] or 0)
    tot += s
    a = agg[lines[i]]
    a[0] += s
    a[1] += float(r[iex] or 0)
    if not a[2]:
        a[2] = r[isrc][:48]
print(f"total stall samples {tot:.0f}")
for k, (s, ex, first) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}%  {k:28s} inst {ex:10.0f}  e.g. {first}")
