#!/bin/bash
# Round-end capture: GPU tests, bench line, launch list, step/level DRAM traffic, ncu --set full
# of the top kernels (each ncu only after the same command ran clean in this call).
set -u
mkdir -p gpurun_out
tools/gpu_check.sh
tools/ncu_traffic.sh > gpurun_out/traffic_run.log 2>&1; echo "traffic rc=$?"
tools/ncu_full.sh ${KERNELS:-k_rowG:2 k_colC:0 k_colA:18 k_rowF:0 k_eqos_bwd:1 k_dyn_bwd:2 k_dyn_fwd:0 k_mr_bwd:0} > gpurun_out/ncu_run.log 2>&1
echo "ncu_full rc=$?"; tail -3 gpurun_out/ncu_run.log
