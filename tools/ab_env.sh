#!/bin/bash
# A/B of runtime switches on the bench workload (under gpurun): tools/ab_env.sh "VAR=a" "VAR=b" ...
# each setting runs bench.py twice (alternating) without the CPU baseline / tree / top-k / CSparse rows
mkdir -p gpurun_out
for rep in 1 2; do
  for s in "$@"; do
    tag=$(echo "$s" | tr ' =' '__')
    env $s timeout 600 python bench.py --no-cpu-baseline --tree-width 0 --topk-keep 0 --csparse-keep 0 \
      > gpurun_out/ab_${tag}_$rep.json 2> gpurun_out/ab_${tag}_$rep.err || tail -3 gpurun_out/ab_${tag}_$rep.err
    python - "$s" gpurun_out/ab_${tag}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:28s} sirius {d['value']:.4f}  dense {d['dense']['ms_per_token']:.4f}  cs {d['cs_only']['ms_per_token']:.4f}  "
      f"verify {d['latency_model']['components_ms']['t_verify']:.3f}  ffn_frac {d['roofline']['frac']:.3f}  clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
  done
done
