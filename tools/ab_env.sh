# Step-rate A/B of an environment switch: bench.py config 2 (no CPU baseline, songs or
# secondary configs) with VAR=a then VAR=b, ROUNDS times; JSON lines in OUT/ab.txt.
# usage: bash tools/ab_env.sh OUT ROUNDS VAR a b [extra bench args]
out=$1; rounds=$2; var=$3; a=$4; b=$5; shift 5
mkdir -p "$out"
for r in $(seq 1 "$rounds"); do
  for v in "$a" "$b"; do
    echo "== $var=$v round $r" >> "$out/ab.txt"
    env "$var=$v" python bench.py --no-cpu-baseline --songs 0 --no-secondary --steps 100 "$@" 2>/dev/null | tail -1 >> "$out/ab.txt"
  done
done
