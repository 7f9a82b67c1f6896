"""Diagnostic: bf16 K/V cache entries written by the GPU prefill vs the oracle's (exact compare):
how many stored elements differ, by how many bf16 ulps, per layer."""
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
cfg = synth.LLAMA3_8B.with_layers(L_) if (len(sys.argv) < 4 or sys.argv[3] != "tiny") else synth.TINY
thr = synth.layer_thresholds(cfg, 0.5)
wh = synth.host_weights(cfg)
MS = P + 64
om = so.OracleModel(cfg, wh, max_seq=MS, max_gamma=16)
prompt = synth.eval_prompt(cfg, 0, P)
first = om.prefill_last(prompt)
ctx = S.Sirius(cfg, sg.device_weights(cfg), thr, batch=1, max_seq=MS, max_gamma=16)
f = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.sirius_prefill(torch.tensor(prompt, dtype=torch.int32, device="cuda"), [P], f)
torch.cuda.synchronize()
KV, hd, L = cfg.n_kv_heads, cfg.head_dim, cfg.n_layers
n = L * KV * MS * hd
for which, name in ((7, "K"), (8, "V")):
    buf = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    S.load().sirius_debug_buffer(ctx.h, 0, which, buf.data_ptr(), n * 2)
    g = buf.float().cpu().numpy().astype(np.float64).reshape(L, KV, MS, hd)[:, :, :P, :]
    for l in range(L):
        k, v = om.read_cache(l, P)
        ref = (k if name == "K" else v).transpose(1, 0, 2)  # [KV, P, hd]
        d = g[l] != ref
        rel = np.abs(g[l] - ref) / np.maximum(np.abs(ref), 1e-30)
        print(f"{name} layer {l}: {int(d.sum())} of {d.size} differ; max rel {rel.max():.2e};"
              f" per position (first 8 differing) {np.unique(np.nonzero(d)[1])[:8].tolist()}", flush=True)
