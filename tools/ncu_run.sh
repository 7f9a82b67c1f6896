#!/bin/bash
# usage: tools/ncu_run.sh <tag>   (run under gpurun) — launch list + full captures of the top kernels
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
# every launch with its device time (cold-cache, serialised): one Sirius kernel after 1 warm-up kernel
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python tools/profile_step.py --kernels 2 > /dev/null 2>&1
# full sections for the top decode kernels (a few launches each, after the prefill + warm-up launches)
for K in ffn_kernel gemv_kernel attn_stage_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -s 200 -c 2 \
    -o gpurun_out/prof_${TAG}_${K} python tools/profile_step.py --kernels 1 > gpurun_out/ncu_${K}.log 2>&1
done
ls -la gpurun_out
