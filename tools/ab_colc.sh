# A/B of the persistent bulk-copy column pass (MGB_COLC_PERSISTENT=1) against the default, plus its parity tests
mkdir -p gpurun_out/r2g
timeout 300 python -m pytest tests -m gpu -q -x -k "conv_level or config1_train or phase_split or kernel_matches" -p no:cacheprovider > gpurun_out/r2g/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest.log
for v in 1 0 1 0; do MGB_COLC_PERSISTENT=$v python tools/step_breakdown.py > gpurun_out/r2g/bd_$v.log 2>&1; cat gpurun_out/r2g/bd_$v.log >> gpurun_out/r2g/ab.txt; echo "persist=$v" >> gpurun_out/r2g/ab.txt; done
MGB_COLC_PERSISTENT=1 python bench.py --no-cpu-baseline --songs 0 > gpurun_out/r2g/bench1.json 2>&1
MGB_COLC_PERSISTENT=0 python bench.py --no-cpu-baseline --songs 0 > gpurun_out/r2g/bench0.json 2>&1
