"""Diagnostic: the float band of the gate activation a = SiLU(g) at Llama-3-8B shapes.

Teacher-forced sparse decode rows on 8B-2L (prompt P): per row and layer, max |a_gpu - a_ref|,
the number of active-set flips, the distance of the nearest |a_ref| to t_l, and the logit error.
Used to size the separation band of the gap-separated thresholds (tests/parity_util.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import synth
from oracle import sirius_oracle as so
from paper_2409_03856_b200 import sirius as S
from synth import gpu as sg

L_ = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P = int(sys.argv[2]) if len(sys.argv) > 2 else 128
N = int(sys.argv[3]) if len(sys.argv) > 3 else 12
cfg = synth.LLAMA3_8B.with_layers(L_)
thr = synth.layer_thresholds(cfg, 0.5)
wh = synth.host_weights(cfg)
om = so.OracleModel(cfg, wh, max_seq=P + N + 32, max_gamma=16)
prompt = synth.eval_prompt(cfg, 0, P)
first = om.prefill_last(prompt)
ctx = S.Sirius(cfg, sg.device_weights(cfg), thr, batch=1, max_seq=P + N + 32, max_gamma=16)
f = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.sirius_prefill(torch.tensor(prompt, dtype=torch.int32, device="cuda"), [P], f)
tok = so.argmax_lowest(first)
Lc, F, V = cfg.n_layers, cfg.ffn_dim, cfg.vocab
for i in range(N):
    ref = om.decode(tok, P + i, True, thr, want_gate=True, want_mask=True)
    to = torch.zeros(1, dtype=torch.int32, device="cuda")
    lo = torch.zeros((1, V), device="cuda")
    na = torch.zeros((1, Lc), dtype=torch.int32, device="cuda")
    ga = torch.zeros((1, Lc, F), device="cuda")
    ctx.sparse_decode_step(torch.tensor([tok], dtype=torch.int32, device="cuda"),
                           torch.tensor([P + i], dtype=torch.int32, device="cuda"), 0, to, lo, na, ga)
    torch.cuda.synchronize()
    g = ga.cpu().numpy()[0]
    e = np.abs(g - ref.gate)
    flips = ((np.abs(g) >= thr[:, None]) != ref.mask.astype(bool)).sum(1)
    near = np.abs(np.abs(ref.gate) - thr[:, None]).min(1)
    le = np.abs(lo.cpu().numpy()[0] - ref.logits).max()
    print(f"row {i}: gate maxerr {[f'{x:.2e}' for x in e.max(1)]} p99 {[f'{x:.1e}' for x in np.quantile(e, 0.99, axis=1)]}"
          f" flips {flips.tolist()} nearest|a|-t {[f'{x:.1e}' for x in near]} logit maxerr {le:.2e}", flush=True)
    tok = so.argmax_lowest(ref.logits)
