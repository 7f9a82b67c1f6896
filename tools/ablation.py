"""Component ablation on the GPU (Table 4 analogue, §5.3; reading D27) and the
SD baseline (greedy-match acceptance, reading D26): Llama-3-8B shape, batch 1, prompt 900, gamma 16,
CATS 50%, r = 0.3 (an operating point where the correction fires).  Per mode: K kernels in a fresh
session; AAL, ms per committed token, tokens that differ from the full model's greedy decode of the same
prompt (the paper measures accuracy; with synthetic weights the closest observable is agreement with
the full model — reported, not asserted).  Writes profiles/ablation_r02.json.

    python tools/ablation.py [--kernels 12] [--r 0.3]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, bench
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

ap = argparse.ArgumentParser()
ap.add_argument("--kernels", type=int, default=12)
ap.add_argument("--r", type=float, default=0.3)
ap.add_argument("--gamma", type=int, default=16)
ap.add_argument("--out", default="profiles/ablation_r02.json")
a = ap.parse_args()
cfg = synth.LLAMA3_8B
w = sg.device_weights(cfg)
thr = synth.layer_thresholds(cfg, 0.5)
prompt = synth.eval_prompt(cfg, 0, 900)
g = a.gamma
ctx = S.Sirius(cfg, w, thr, batch=1, max_seq=900 + (a.kernels + 4) * g + 64, max_gamma=g)
n_tok = a.kernels * g
# the full model's greedy continuation (reference for agreement)
dd = driver.Driver(ctx)
ref = dd.greedy([prompt], n_tok + 1, dense=True).tokens[0]
modes = {"sirius (rewrite + interleave + rollback)": dict(rewrite=True, interleave=True, rollback=True),
         "interleave only": dict(rewrite=False, interleave=True, rollback=False),
         "KV rewrite only": dict(rewrite=True, interleave=False, rollback=False),
         "rewrite + interleave": dict(rewrite=True, interleave=True, rollback=False),
         "interleave + rollback (no rewrite)": dict(rewrite=False, interleave=True, rollback=True),
         "no correction (sparse only)": None}
res = {}
clk = bench.Clocks(0)
clk.start()
st = torch.cuda.current_stream()
for name, m in modes.items():
    if m is None:
        toks = driver.Driver(ctx).greedy([prompt], n_tok + 1, dense=False).tokens[0]
        res[name] = {"agree_with_full": float(np.mean(np.array(toks[:n_tok]) == np.array(ref[:n_tok])))}
        continue
    drv = driver.Driver(ctx, **m)
    drv.begin([prompt])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    adv = [drv.step(g, a.r) for _ in range(a.kernels)]
    e1.record(st)
    torch.cuda.synchronize()
    drv.flush()
    toks = drv.out[0][:n_tok]
    nn = min(len(toks), len(ref))
    res[name] = {"aal": float(np.mean(adv)), "ms_per_token": e0.elapsed_time(e1) / sum(adv),
                 "agree_with_full": float(np.mean(np.array(toks[:nn]) == np.array(ref[:nn]))),
                 "rejections": int(sum(1 for k in drv.log if int(k.j[0]) < g - 1))}
drv = driver.Driver(ctx)
drv.begin([prompt])
adv = [drv.step(g, 0.0, S.ACCEPT_EXACT_ARGMAX) for _ in range(a.kernels)]
drv.flush()
nn = min(len(drv.out[0]), n_tok)
res["SD greedy match (lossless)"] = {"aal": float(np.mean(adv)),
                                     "agree_with_full": float(np.mean(np.array(drv.out[0][:nn]) == np.array(ref[:nn])))}
out = {"config": f"llama3-8b shape, batch 1, prompt 900, gamma {g}, CATS 0.5, r {a.r}, {a.kernels} kernels per mode",
       "modes": res, "clocks": clk.stop()}
print(json.dumps(out, indent=1))
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(out, f, indent=1)
