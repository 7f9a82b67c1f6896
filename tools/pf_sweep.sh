#!/bin/bash
# L2-prefetch plan sweep (run under gpurun): bench.py per setting, one summary line each
mkdir -p gpurun_out
run() {
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 6 > gpurun_out/sweep_tmp.json 2>gpurun_out/sweep_err.log
  python - "$*" <<'PY'
import json, sys
try:
    r = json.loads(open("gpurun_out/sweep_tmp.json").read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open("gpurun_out/sweep_err.log").read()[-800:]); sys.exit()
k = r["per_kernel_device_ms"]
per = lambda n: k.get(n, {"ms_total": 0, "launches": 0})["ms_total"] / max(k.get(n, {"launches": 1})["launches"], 1) * 1e3
print(f"{sys.argv[1]:45s} sirius {r['value']:.3f} dense {r['dense']['ms_per_token']:.3f} cs {r['cs_only']['ms_per_token']:.3f} "
      f"roof {r['roofline']['frac']:.3f} | qkv {per('qkv_gemv'):.1f} attn {per('attn_decode'):.1f} o {per('oproj_gemv'):.1f} ffn {per('cats_ffn'):.1f} "
      f"head {per('lm_head'):.1f} step {per('decode_step'):.1f} corr {per('correct_kernel'):.0f} us  aal {r['sirius']['aal']:.2f} sm {r['clocks']['sm_mhz']}")
PY
}
for spec in "$@"; do run $spec; done
