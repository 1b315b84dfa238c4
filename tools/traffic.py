"""Per-kernel DRAM traffic and time of the last full train step in an ncu metrics CSV
(tools/ncu_traffic.sh).  Prints a table and writes a JSON summary next to the CSV."""
import collections
import csv
import json
import re
import sys

path = sys.argv[1]
level = sys.argv[sys.argv.index("--level") + 1] if "--level" in sys.argv else None
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
per = int(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 0
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
# one row per (launch, metric): group by launch ID
launches = collections.OrderedDict()
for d in data:
    key = d["ID"]
    L = launches.setdefault(key, {"name": re.sub(r"\(.*", "", d["Kernel Name"]), "grid": d.get("Grid Size", "")})
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    if d["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        L[d["Metric Name"]] = v * scale
    elif d["Metric Name"].startswith("sm__"):  # FP32 (FMA pipe) / issue utilisation, % of peak
        L[d["Metric Name"]] = v
    else:
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        L["us"] = v * scale
lst = list(launches.values())
if level:  # --profile-level run: the last reps x per launches are the level's fwd+bwd repetitions
    step = lst[-reps * per:]
else:
    ends = [i for i, L in enumerate(lst) if "k_optim_step" in L["name"]] or \
        [i for i, L in enumerate(lst) if "k_project" in L["name"]]
    step = lst[ends[-2] + 1: ends[-1] + 1] if len(ends) >= 2 else lst
tot_b = sum(L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0) for L in step)
tot_t = sum(L.get("us", 0) for L in step)
print(f"launches {len(step)}  DRAM {tot_b / 1e9:.3f} GB  serialised {tot_t / 1e3:.3f} ms  "
      f"avg {tot_b / (tot_t * 1e-6) / 1e12:.2f} TB/s")
FMA = "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"
ISSUE = "sm__inst_issued.avg.pct_of_peak_sustained_active"
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for L in step:
    a = agg[L["name"][:60]]
    a[0] += 1
    a[1] += L.get("us", 0)
    a[2] += L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    a[3] += L.get(FMA, 0) * L.get("us", 0)  # time-weighted utilisations
    a[4] += L.get(ISSUE, 0) * L.get("us", 0)
print("      time    n       DRAM    HBM    FP32-FMA  issue  kernel")
for k, (n, us, b, f, i) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:8.1f} us x{n:2d}  {b / 1e6:8.1f} MB  {b / (us * 1e-6) / 1e12 if us else 0:5.2f} TB/s"
          f"  {f / us if us else 0:5.1f} %  {i / us if us else 0:5.1f} %  {k}")
out = {"launches": step, "dram_bytes_step": tot_b, "serialised_us": tot_t}
if level:
    out = {"level": level, "reps": reps, "dram_bytes_per_rep": tot_b / reps, "serialised_us_per_rep": tot_t / reps,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold, serialised)",
           "launches": step}
    print(f"level {level}: {tot_b / reps / 1e6:.1f} MB DRAM per fwd+bwd, {tot_t / reps:.1f} us serialised")
json.dump(out, open(path.replace(".csv", ".json"), "w"), indent=1)
