# A/B of the EQ FIR synthesis / adjoint as float64 table products (default) vs rotation recurrences (MGB_EQ_FIR_MM=0)
mkdir -p gpurun_out/eqf
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "kernel_matches or conv_level or config1 or config2_train or phase_split or reference_tape or batched_training" > gpurun_out/eqf/pytest.log 2>&1; echo rc=$? >> gpurun_out/eqf/pytest.log
for v in 1 0 1 0; do
  MGB_EQ_FIR_MM=$v python tools/batch_step_profile.py > gpurun_out/eqf/bp_$v.json 2>&1
  MGB_EQ_FIR_MM=$v python tools/step_breakdown.py > gpurun_out/eqf/bd_$v.json 2>&1
  echo "mm=$v $(tail -1 gpurun_out/eqf/bp_$v.json) $(tail -1 gpurun_out/eqf/bd_$v.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fir_synthesis"], d["captured_step_ms"])')" >> gpurun_out/eqf/ab.txt
done
