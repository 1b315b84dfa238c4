"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: the last full train step."""
import collections
import csv
import re
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
# one train step ends with the optimiser pass (k_optim_step; k_project / k_adamw in
# captures of earlier builds)
ends = [i for i, d in enumerate(data) if "k_optim_step" in d["Kernel Name"]] or \
    [i for i, d in enumerate(data) if "k_project" in d["Kernel Name"]] or \
    [i for i, d in enumerate(data) if "k_adamw" in d["Kernel Name"]]
if len(ends) >= 2:
    step = data[ends[-2] + 1: ends[-1] + 1]
else:
    n = len(data) // steps
    step = data[-n:]
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for d in step:
    name = re.sub(r"\(.*", "", d["Kernel Name"])[:70]
    t = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
    agg[name][0] += 1
    agg[name][1] += t
    tot += t
print(f"launches in one step: {len(step)}, total {tot:.3f} ms (serialised, cold)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1]:8.3f} ms {100 * v[1] / tot:5.1f}%  x{v[0]:3d}  {k}")

if len(sys.argv) > 3 and sys.argv[3] == "seq":
    print("--- launch sequence of the last step")
    for d in step:
        name = re.sub(r"\(.*", "", d["Kernel Name"])[:60]
        t = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        print(f"{1000 * t:9.1f} us  grid={d.get('Grid Size', '?'):>16}  {name}")
