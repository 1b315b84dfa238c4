# Step-rate A/B of library builds (tools/bin/<name>.so): bench.py config 2 without the
# CPU baseline, songs or secondary configs; one JSON line per run in OUT/ab.txt.
# usage: bash tools/ab_step.sh OUT ROUNDS name1 name2 ...
out=$1; rounds=$2; shift 2
bash tools/ab_lib.sh "$out" "$rounds" "python bench.py --no-cpu-baseline --songs 0 --no-secondary --steps 100 2>/dev/null | tail -1" "$@"
