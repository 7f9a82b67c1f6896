"""Profiling driver (for ncu): Llama-3-8B shape, prompt P, a few Sirius kernels (sparse decode steps
+ correct_kernel + kv_rewrite).  Not a benchmark: numbers printed here are not bench values."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--prompt", type=int, default=900)
ap.add_argument("--kernels", type=int, default=2)
ap.add_argument("--gamma", type=int, default=16)
a = ap.parse_args()
cfg = synth.CONFIGS[a.model]
w = sg.device_weights(cfg)
ctx = S.Sirius(cfg, w, synth.layer_thresholds(cfg, 0.5), batch=1, max_seq=a.prompt + 64 * a.gamma, max_gamma=a.gamma)
drv = driver.Driver(ctx)
drv.begin([synth.eval_prompt(cfg, 0, a.prompt)])
for _ in range(a.kernels):
    drv.step(a.gamma, 0.1)
drv.flush()
torch.cuda.synchronize()
print("done", drv.T)
