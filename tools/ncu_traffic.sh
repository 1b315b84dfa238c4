#!/bin/bash
# DRAM bytes + duration of every launch of one eager config-2 step (ncu, cold, serialised).
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/traffic.csv python bench.py --eager-profile 1 > gpurun_out/traffic.log 2>&1
echo "ncu=$?"
python tools/traffic.py gpurun_out/traffic.csv > gpurun_out/traffic.txt; head -60 gpurun_out/traffic.txt
