"""Phase timeline of the per-stage CATS FFN kernel of one decode layer (Llama-3-8B shape; globaltimer
stamps per CTA, debug path, not a benchmark)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

cfg = synth.CONFIGS["llama3-8b"]
ctx = S.Sirius(cfg, sg.device_weights(cfg), synth.layer_thresholds(cfg, 0.5), batch=1, max_seq=1200, max_gamma=16)
drv = driver.Driver(ctx)
drv.begin([synth.eval_prompt(cfg, 0, 900)])
ctx.graphs(False)
buf = torch.zeros((8, 1024), dtype=torch.int64, device="cuda")
tok = torch.tensor([drv.pending[0]], dtype=torch.int32, device="cuda")
out = torch.zeros(1, dtype=torch.int32, device="cuda")
for i in range(3):
    buf.zero_()
    assert ctx.lib.sirius_debug_trace_ffn(ctx.h, buf.data_ptr(), 7) == 0
    ctx.sparse_decode_step(tok, torch.tensor([900 + i], dtype=torch.int32, device="cuda"), 0, out)
    torch.cuda.synchronize()
ctx.lib.sirius_debug_trace_ffn(ctx.h, None, -1)
t = buf.cpu().numpy().astype(np.float64)
ok = t[0] != 0
t = (t[:, ok] - t[0, ok].min()) / 1e3
print(f"CTAs {ok.sum()}  span {t[6].max():.2f} us  start spread {t[0].max() - t[0].min():.2f}  end spread {t[6].max() - t[6].min():.2f}")
for k, n in enumerate(["prologue", "gate rows", "ballot", "up rows", "down rows", "atomics out"]):
    d = t[k + 1] - t[k]
    print(f"{n:12s} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  max {d.max():6.2f}")
starts = np.sort(t[0])
print("CTA start times (us): first 5", starts[:5].round(2), "last 5", starts[-5:].round(2))
