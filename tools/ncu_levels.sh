#!/bin/bash
# DRAM bytes of every conv (and scan) level's forward+backward at config 2, one ncu
# metrics capture per level (cold caches, serialised), merged into
# gpurun_out/level_traffic_config2.json for bench.py's roofline.traffic; then the
# step's launch list and one `ncu --set full` capture of the top kernels.
mkdir -p gpurun_out/lv
for LEVEL in ${LEVELS:-r@step7 d@step6 e@step1 c@step2 n@step3 r@step15 d@step14 e@step9}; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/lv/$LEVEL.csv python bench.py --eager-profile 3 --profile-level "$LEVEL" \
    > gpurun_out/lv/$LEVEL.log 2>&1
  PER=$(python -c "import json; print([json.loads(l) for l in open('gpurun_out/lv/$LEVEL.log') if l.startswith('{\"profile_level')][-1]['launches_per_rep'])")
  python tools/traffic.py gpurun_out/lv/$LEVEL.csv --level "$LEVEL" --reps 3 --per "$PER" > gpurun_out/lv/$LEVEL.txt
  echo "$LEVEL: $(tail -1 gpurun_out/lv/$LEVEL.txt)"
done
python - <<'PY'
import glob, json
out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum (cold, serialised; "
                 "tools/ncu_levels.sh): one level's forward + backward, bench.py --eager-profile 3 --profile-level",
       "levels": {}}
for f in sorted(glob.glob("gpurun_out/lv/*.json")):
    d = json.load(open(f))
    out["levels"][d["level"]] = {"dram_bytes_per_rep": d["dram_bytes_per_rep"],
                                 "serialised_us_per_rep": d["serialised_us_per_rep"]}
json.dump(out, open("gpurun_out/level_traffic_config2.json", "w"), indent=1)
print(json.dumps(out["levels"], indent=0))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --eager-profile 2 > gpurun_out/launches.log 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launch_list.txt 2>&1
bash tools/ncu_full.sh k_rowG:1 k_colC:3 k_rowF:1 k_colA:4 k_dyn_bwd:1 k_mr_bwd:1 > gpurun_out/ncu_full.log 2>&1
