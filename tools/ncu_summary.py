"""Summarise an ncu report: key metrics, instruction mix, top stall sites."""
import csv
import io
import subprocess
import sys
from collections import Counter


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=30):
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    want = ("Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Achieved Occupancy",
            "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
            "Compute (SM) Throughput", "DRAM Throughput", "Waves Per SM")
    for r in det[1:]:
        if len(r) > 14 and r[-4] in want:
            print(f"{r[-4]:40s} {r[-2]:>14s} {r[-3]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
    for k, x in zip(h, v):
        if ("average_warps_issue_stalled" in k and "per_issue_active" in k and x not in ("", "0")) or \
           k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
                 "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
            print(f"{k:80s} {x}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hh = src[1]
    data = src[2:]
    isrc, iss, iex = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    c = Counter()
    for r in data:
        t = r[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op.split(".")[0]] += float(r[iex] or 0)
    print("instruction mix:", c.most_common(16))
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:top]:
        print(f"{r[iss]:>8s} {r[iex]:>10s}  {r[isrc][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
