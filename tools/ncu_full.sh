#!/bin/bash
# One `ncu --set full` capture per kernel name (one launch each) of an eager
# config-2 step.  Exports the details page and raw metrics as text/CSV on the
# box (gpurun_out/ncu_<name>.{txt,csv}, hottest source lines in _lines.txt); the
# .ncu-rep is kept only with KEEP=1.  NCU_BASE=demangled matches template arguments.
# usage: tools/ncu_full.sh name[:skip] ...   (skip = matching launches to skip)
mkdir -p gpurun_out
for spec in "$@"; do
  k=${spec%%:*}; skip=0
  [[ "$spec" == *:* ]] && skip=${spec##*:}
  tag=${TAG:-$(echo "$k" | tr -c 'A-Za-z0-9_\n' '_' | cut -c1-24)}
  rep=/tmp/ncu_${tag}_${skip}
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base ${NCU_BASE:-function} -k "regex:$k" --launch-skip "$skip" -c 1 \
    -o "$rep" -f ${NCU_CMD:-python bench.py --eager-profile 1} > "gpurun_out/ncu_${tag}.log" 2>&1
  echo "$k rc=$?"
  ncu -i "$rep.ncu-rep" --page details > "gpurun_out/ncu_${tag}_${skip}.txt" 2>&1
  ncu -i "$rep.ncu-rep" --page raw --csv > "gpurun_out/ncu_${tag}_${skip}_raw.csv" 2>&1
  ncu -i "$rep.ncu-rep" --page source --csv 2>&1 | gzip > "gpurun_out/ncu_${tag}_${skip}_src.csv.gz"
  python tools/ncu_lines.py "$rep.ncu-rep" 45 > "gpurun_out/ncu_${tag}_${skip}_lines.txt" 2>&1
  [ "${KEEP:-0}" = 1 ] && cp "$rep.ncu-rep" gpurun_out/
done
du -sh gpurun_out
