#!/bin/bash
# GPU round trip: parity tests, bench (JSON line), ncu launch list of one eager step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; rc=$?; echo "bench=$rc"; tail -1 gpurun_out/bench.log
if [ "$rc" = 0 ] && [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --eager-profile 1 > gpurun_out/ncu.log 2>&1; echo "ncu=$?"
  python tools/launches.py gpurun_out/launches.csv > gpurun_out/launch_list.txt; head -40 gpurun_out/launch_list.txt
fi
