#!/bin/bash
# Per-rank TP compute proxies (tools/tp_proxy.py) for BASELINE configs[2] / [3] on one GPU -> profiles/
mkdir -p gpurun_out
# usage: tools/run_proxies.sh [--par]   (--par: decode all-reduces fused, looped back on-chip)
PAR=${1:-}
SUF=${PAR:+_par}
for spec in "llama3-8b 2 1" "llama3-8b 4 1" "llama3-8b 8 1" "llama3-8b 8 8" "llama3-70b 8 1"; do
  set -- $spec
  timeout 900 python tools/tp_proxy.py --model $1 --tp $2 --batch $3 $PAR --out gpurun_out/tp_proxy_$1_tp$2_b$3$SUF.json \
    > gpurun_out/tp_proxy_$1_tp$2_b$3$SUF.log 2>&1 || tail -5 gpurun_out/tp_proxy_$1_tp$2_b$3$SUF.log
  tail -1 gpurun_out/tp_proxy_$1_tp$2_b$3$SUF.log | cut -c1-400
done
