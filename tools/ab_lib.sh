# A/B of library builds on one box: for each round, each tools/bin/<name>.so in turn is
# installed as the package library and "cmd" runs; output appended to OUT/ab.txt.
# usage: bash tools/ab_lib.sh OUT ROUNDS "cmd" name1 name2 ...
out=$1; rounds=$2; cmd=$3; shift 3
mkdir -p "$out"
lib=paper_2509_15948_b200/libmixgraph_b200.so
cp "$lib" "$out/.lib_saved.so"
for r in $(seq 1 "$rounds"); do
  for name in "$@"; do
    cp "tools/bin/$name.so" "$lib"
    echo "== $name round $r" >> "$out/ab.txt"
    bash -c "$cmd" >> "$out/ab.txt" 2>&1
  done
done
cp "$out/.lib_saved.so" "$lib"
rm -f "$out/.lib_saved.so"
