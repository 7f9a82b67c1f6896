"""Launch list of top-k FSparse decode steps (for ncu --metrics gpu__time_duration.sum): Llama-3-8B
shape, prompt 900, 4 greedy top-k steps after 2 warm-up steps.  Not a benchmark."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

cfg = synth.CONFIGS["llama3-8b"]
ctx = S.Sirius(cfg, sg.device_weights(cfg), synth.layer_thresholds(cfg, 0.5), batch=1, max_seq=1200, max_gamma=16)
ctx.sirius_topk_enable(0.5)
drv = driver.Driver(ctx, topk=True)
drv.begin([synth.eval_prompt(cfg, 0, 900)])
drv.greedy_run(drv.pending, drv.T, 2, False)
drv.greedy_run(drv.pending, [t + 2 for t in drv.T], 4, False)
torch.cuda.synchronize()
print("done")
