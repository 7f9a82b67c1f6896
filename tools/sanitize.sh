#!/bin/bash
# compute-sanitizer passes over the tiny-config smoke run (prefill, sparse decode, correct_kernel,
# kv_rewrite, the CATS / dense / persistent paths through the graphs) — SURVEY.md §4 T5.  Run under
# gpurun; logs in gpurun_out/sanitize_*.log, one summary line each.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  SIRIUS_GRAPHS=1 timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|smoke ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
