"""Summarise gpurun_out/ncu_<k>_<skip>{.txt,_raw.csv,_src.csv.gz}: headline metrics, stall mix, hottest SASS."""
import csv
import gzip
import re
import sys

for tag in sys.argv[1:]:
    txt = open(f"gpurun_out/ncu_{tag}.txt").read()
    print("==", tag, re.search(r"\((\d+), (\d+), (\d+)\)x\((\d+), 1, 1\)", txt).group(0))
    for key in ["Duration", "DRAM Throughput", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
                "Issue Slots Busy", "Eligible Warps Per Scheduler", "Dynamic Shared Memory Per Block", "L2 Hit Rate"]:
        m = re.search(r"^\s+" + re.escape(key) + r"\s+(\S+)\s+([\d.,]+)", txt, re.M)
        if m:
            print(f"   {key}: {m.group(2)} {m.group(1)}")
    rows = list(csv.reader(open(f"gpurun_out/ncu_{tag}_raw.csv")))
    h, v = rows[0], rows[2]
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in x:
            try:
                st.append((x.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i].replace(",", ""))))
            except ValueError:
                pass
    st.sort(key=lambda t: -t[1])
    tot = sum(b for _, b in st) or 1
    print("   stalls:", ", ".join(f"{a} {100*b/tot:.0f}%" for a, b in st[:6]))
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]:
        if key in h:
            i = h.index(key)
            print(f"   {key}: {v[i]} {rows[1][i]}")
    try:
        src = list(csv.reader(gzip.open(f"gpurun_out/ncu_{tag}_src.csv.gz", "rt")))
    except FileNotFoundError:  # the hottest source lines are in ncu_<tag>_lines.txt instead
        continue
    hdr, src = src[1], src[2:]
    src = [r for r in src if len(r) > 2 and r[2].isdigit()]
    tot = sum(int(r[2]) for r in src) or 1
    top = sorted(range(len(src)), key=lambda i: -int(src[i][2]))[:int(sys.argv[0] and 8)]
    for i in sorted(top):
        print(f"   {i:5d} {100*int(src[i][2])/tot:4.1f}% {src[i][1].strip()[:70]}")
