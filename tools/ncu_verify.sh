#!/bin/bash
# full ncu captures of the verify-path kernels of verify layer 0 (skipping the 900-token prefill:
# 4 chunks x 32 layers of attn_rows / 4 GEMMs each)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_rows_kernel -s 128 -c 1 \
  -o gpurun_out/prof_${TAG}_attn_rows python tools/profile_step.py --kernels 1 > gpurun_out/ncu_attn_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1024 -c 4 \
  -o gpurun_out/prof_${TAG}_gemm_verify python tools/profile_step.py --kernels 1 > gpurun_out/ncu_gemm_verify.log 2>&1
ls -la gpurun_out | tail -5
