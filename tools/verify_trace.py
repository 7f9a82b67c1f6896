"""Phase timeline of the verify attention (attn_rows_kernel) of one layer, Llama-3-8B shape, gamma 16,
900-token context (globaltimer stamps per CTA; debug path, not a benchmark)."""
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
buf = torch.zeros((5, 8, 1024), dtype=torch.int64, device="cuda")  # attn_rows, then QKV / O / gate-up / down GEMMs
for rep in range(3):
    buf.zero_()
    assert ctx.lib.sirius_debug_trace_verify(ctx.h, buf.data_ptr(), 5) == 0
    drv.step(16, 0.1)
    torch.cuda.synchronize()
ctx.lib.sirius_debug_trace_verify(ctx.h, None, -1)
allb = buf.cpu().numpy().astype(np.float64)
t = allb[0][:, :1024]
ok = t[0] != 0
t = (t[:, ok] - t[0, ok].min()) / 1e3
names = ["q load", "K/V block load", "scores", "softmax+PV", "partial write", "group barrier", "combine"]
print(f"CTAs {ok.sum()}  kernel span {t[7].max():.2f} us (first start -> last end); start spread {t[0].max() - t[0].min():.2f}")
for k, n in enumerate(names):
    d = t[k + 1] - t[k]
    print(f"{n:16s} median {np.median(d):6.2f}  max {d.max():6.2f} us")

gn = ["QKV", "O-proj", "gate+up", "down"]
stage = ["start->setup", "setup->pdl wait done", "wait->first stage landed", "first stage->1st accum", "1st accum->all done"]
for gi in range(4):
    g = allb[1 + gi][:6, :1024]
    ok = g[0] != 0
    if not ok.any():
        continue
    g = (g[:, ok] - g[0, ok].min()) / 1e3
    print(f"GEMM {gn[gi]}: span {g[5].max():.2f} us, start spread {g[0].max():.2f}")
    for k, n in enumerate(stage):
        d = g[k + 1] - g[k]
        print(f"   {n:26s} median {np.median(d):6.2f}  max {d.max():6.2f}")
