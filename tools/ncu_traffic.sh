#!/bin/bash
# DRAM bytes + duration of every launch of one eager config-2 step, and of the
# dominant level alone (ncu metrics; cold caches, serialised).
mkdir -p gpurun_out
LEVEL=${LEVEL:-d@step6}
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none \
  --csv --log-file gpurun_out/traffic.csv python bench.py --eager-profile 1 > gpurun_out/traffic.log 2>&1
echo "ncu step=$?"
python tools/traffic.py gpurun_out/traffic.csv > gpurun_out/traffic.txt; head -30 gpurun_out/traffic.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/level_traffic.csv python bench.py --eager-profile 3 --profile-level "$LEVEL" \
  > gpurun_out/level_traffic.log 2>&1
echo "ncu level=$?"
PER=$(python -c "import json,sys; print([json.loads(l) for l in open('gpurun_out/level_traffic.log') if l.startswith('{\"profile_level')][-1]['launches_per_rep'])")
python tools/traffic.py gpurun_out/level_traffic.csv --level "$LEVEL" --reps 3 --per "$PER" > gpurun_out/level_traffic.txt
cat gpurun_out/level_traffic.txt
