"""Ad-hoc GPU-vs-oracle stage diagnostics (tiny config)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from synth import gpu as sg
from oracle import sirius_oracle as so
from paper_2409_03856_b200 import sirius as S

cfg = synth.TINY
wh = synth.host_weights(cfg); wd = sg.device_weights(cfg)
thr = synth.layer_thresholds(cfg, 0.5)
def ctx(): return S.Sirius(cfg, wd, thr, batch=1, max_seq=256, max_gamma=16)
def dec(c, tok, pos, flags=S.SIRIUS_DENSE):
    lo = torch.zeros((1, cfg.vocab), device="cuda"); to = torch.zeros(1, dtype=torch.int32, device="cuda")
    c.sparse_decode_step(torch.tensor([tok], dtype=torch.int32, device="cuda"), torch.tensor([pos], dtype=torch.int32, device="cuda"), flags, to, lo)
    torch.cuda.synchronize(); return lo.cpu().numpy()[0]
# 1: decode at pos 0..5 from empty cache
c = ctx(); om = so.OracleModel(cfg, wh, max_seq=256)
toks = synth.eval_prompt(cfg, 0, 8)
for p in range(6):
    g = dec(c, int(toks[p]), p); r = om.decode(int(toks[p]), p, False).logits
    print("decode pos", p, "maxerr", np.abs(g - r).max())
# 2: verify from T=0 with gamma=6 on a fresh ctx
c2 = ctx(); om2 = so.OracleModel(cfg, wh, max_seq=256)
kt = torch.tensor([toks[:6]], dtype=torch.int32, device="cuda"); st = torch.zeros(1, dtype=torch.int32, device="cuda")
na = torch.zeros(1, dtype=torch.int32, device="cuda"); nx = torch.zeros(1, dtype=torch.int32, device="cuda")
lo = torch.zeros((1, 6, cfg.vocab), device="cuda")
c2.correct_kernel(kt, st, 6, 0.1, 0, na, nx, None, lo); torch.cuda.synchronize()
lf = om2.verify([int(t) for t in toks[:6]], 0)
print("verify T=0 maxerr per row", np.abs(lo.cpu().numpy()[0] - lf).max(1))
# 3: prefill 6 then decode pos 6
c3 = ctx(); om3 = so.OracleModel(cfg, wh, max_seq=256)
first = torch.zeros(1, dtype=torch.int32, device="cuda")
c3.sirius_prefill(torch.tensor(toks[:6], device="cuda"), [6], first); torch.cuda.synchronize()
ref = om3.prefill(toks[:6])
print("prefill first", first.item(), so.argmax_lowest(ref[-1]))
g = dec(c3, int(toks[6]), 6); r = om3.decode(int(toks[6]), 6, False).logits
print("decode after prefill maxerr", np.abs(g - r).max())
# 4: sparse decode from empty cache
c4 = ctx(); om4 = so.OracleModel(cfg, wh, max_seq=256)
for p in range(3):
    g = dec(c4, int(toks[p]), p, 0); r = om4.decode(int(toks[p]), p, True, thr).logits
    print("sparse decode pos", p, "maxerr", np.abs(g - r).max())
