#!/bin/bash
# full ncu captures of the verify-path kernels (skipping the prefill launches)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_rows_kernel -s 132 -c 1 \
  -o gpurun_out/prof_${TAG}_attn_rows python tools/profile_step.py --kernels 1 > gpurun_out/ncu_attn_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 516 -c 4 \
  -o gpurun_out/prof_${TAG}_gemm_verify python tools/profile_step.py --kernels 1 > gpurun_out/ncu_gemm_verify.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:norm_rows_kernel -s 260 -c 1 \
  -o gpurun_out/prof_${TAG}_norm_rows python tools/profile_step.py --kernels 1 > gpurun_out/ncu_norm_rows.log 2>&1
ls -la gpurun_out | tail -5
