"""Diagnostic: TP-emulated decode (tp = 2, 8) against TP 1 on the GPU and the oracle, per stage."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from synth import gpu as sg
from oracle import sirius_oracle as so
from paper_2409_03856_b200 import sirius as S

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
P = int(sys.argv[2]) if len(sys.argv) > 2 else 17
thr = synth.layer_thresholds(cfg, 0.5)
wh = synth.host_weights(cfg)
om = so.OracleModel(cfg, wh, max_seq=256, max_gamma=16)
prompt = synth.eval_prompt(cfg, 3, P)
first = om.prefill_last(prompt)
tok = so.argmax_lowest(first)
ref = om.decode(tok, P, True, thr, want_gate=True, want_mask=True)
L, F, V = cfg.n_layers, cfg.ffn_dim, cfg.vocab
for tp in (1, 2, 8):
    if cfg.n_kv_heads % tp:
        continue
    w = sg.device_weights(cfg) if tp == 1 else [sg.device_weights(cfg, tp, r) for r in range(tp)]
    ctx = S.Sirius(cfg, w, thr, batch=1, max_seq=256, max_gamma=16, tp_size=tp)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(torch.tensor(prompt, dtype=torch.int32, device="cuda"), [P], f)
    to = torch.zeros(1, dtype=torch.int32, device="cuda")
    lo = torch.zeros((1, V), device="cuda")
    na = torch.zeros((1, L), dtype=torch.int32, device="cuda")
    ga = torch.zeros((1, L, F), device="cuda")
    ctx.sparse_decode_step(torch.tensor([tok], dtype=torch.int32, device="cuda"),
                           torch.tensor([P], dtype=torch.int32, device="cuda"), 0, to, lo, na, ga)
    torch.cuda.synchronize()
    g = ga.cpu().numpy()[0]
    e = np.abs(g - ref.gate)
    rel = e / (1e-3 + np.abs(ref.gate))
    print(f"tp={tp} first {int(f.item())}/{so.argmax_lowest(first)} logits maxerr {np.abs(lo.cpu().numpy()[0] - ref.logits).max():.3e}"
          f" gate maxerr per layer {[float(x) for x in e.max(1)]} worst rel {[float(x) for x in rel.max(1)]}"
          f" at {[int(x) for x in rel.argmax(1)]} n_active {na.cpu().numpy()[0].tolist()} ref {ref.n_active.tolist()}")
    del ctx
