"""Hottest CUDA source lines of an ncu report (stall samples and instructions per line).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = "?", [], None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        samp, inst = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    rows.append((samp, inst, fname, r[0], r[1].strip()))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"samples {ts:.0f} instructions {ti:.0f}")
for samp, inst, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100*samp/ts:5.1f}% smp {100*inst/ti:5.1f}% ins  {f}:{ln}  {src[:90]}")
