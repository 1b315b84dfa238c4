#!/bin/bash
# A/B the built library against experiment builds in paper_2509_15948_b200/variants/*.so:
# quick parity subset + bench per variant (the box copy of the library is swapped in place).
mkdir -p gpurun_out
LIB=paper_2509_15948_b200/libmixgraph_b200.so
cp $LIB /tmp/base.so
for v in base paper_2509_15948_b200/variants/*.so; do
  name=$(basename $v .so)
  if [ "$v" = base ]; then cp /tmp/base.so $LIB; else cp $v $LIB; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${AB_TESTS:-conv or golden or train_step}" > gpurun_out/ab_pytest_$name.log 2>&1
  echo "$name pytest=$? $(tail -1 gpurun_out/ab_pytest_$name.log)"
  for rep in 1 2; do
    timeout 300 python bench.py --steps 40 --warmup 5 --e2e-steps 4 > gpurun_out/ab_bench_${name}_$rep.log 2>&1
    python - gpurun_out/ab_bench_${name}_$rep.log $name <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); lv=d["levels_ms"]
print("  %-8s value=%.1f trial=%.3f " % (sys.argv[2], d["value"], d.get("eval_trial_ms", 0)) + " ".join("%s=%.4f" % (k.split("@")[0]+k.split("B=")[1][:-1], v) for k, v in lv.items()))
PY
  done
done
cp /tmp/base.so $LIB
