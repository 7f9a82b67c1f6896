#!/bin/bash
# round-end ncu pass (under gpurun): launch list + full captures, summarised ON the box so that
# gpurun_out stays under the copy-back limit (only the FFN report is kept).
TAG=${1:-r01}
bash tools/ncu_run.sh $TAG > gpurun_out/ncu_run.log 2>&1
bash tools/ncu_verify.sh $TAG > gpurun_out/ncu_verify.log 2>&1
python tools/ncu_summary.py $TAG gpurun_out/prof_${TAG}_ffn_kernel.ncu-rep gpurun_out/prof_${TAG}_gemv_kernel.ncu-rep \
  gpurun_out/prof_${TAG}_attn_stage_kernel.ncu-rep gpurun_out/prof_${TAG}_gemm_verify.ncu-rep \
  gpurun_out/prof_${TAG}_attn_rows.ncu-rep > gpurun_out/ncu_summary_${TAG}.txt 2>&1
cp profiles/ncu_summary_${TAG}.json gpurun_out/
python tools/launch_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/${TAG}_launch_summary.txt
gzip -f gpurun_out/launches_${TAG}.csv
rm -f gpurun_out/prof_${TAG}_gemv_kernel.ncu-rep gpurun_out/prof_${TAG}_attn_stage_kernel.ncu-rep \
  gpurun_out/prof_${TAG}_gemm_verify.ncu-rep gpurun_out/prof_${TAG}_attn_rows.ncu-rep
du -sh gpurun_out
