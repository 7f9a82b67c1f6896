"""Diagnostic: where the decode row's float error comes from (8B-1L, one sparse decode row after a
dense prefill).  Every GPU intermediate is compared with an fp64 numpy recomputation of that stage
from the GPU's own inputs to the stage (isolates each kernel), and the attention is also recomputed
on the oracle's K/V cache (the effect of bf16 K/V rounding flips)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import synth
from oracle import sirius_oracle as so
from paper_2409_03856_b200 import sirius as S
from synth import gpu as sg

P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = synth.LLAMA3_8B.with_layers(1)
thr = synth.layer_thresholds(cfg, 0.5)
wh = synth.host_weights(cfg)
MS = P + 64
om = so.OracleModel(cfg, wh, max_seq=MS, max_gamma=16)
prompt = synth.eval_prompt(cfg, 0, P)
tok = so.argmax_lowest(om.prefill_last(prompt))
ctx = S.Sirius(cfg, sg.device_weights(cfg), thr, batch=1, max_seq=MS, max_gamma=16)
f = torch.zeros(1, dtype=torch.int32, device="cuda")
ctx.sirius_prefill(torch.tensor(prompt, dtype=torch.int32, device="cuda"), [P], f)
ref = om.decode(tok, P, True, thr, want_gate=True)
ga = torch.zeros((1, 1, cfg.ffn_dim), device="cuda")
lo = torch.zeros((1, cfg.vocab), device="cuda")
ctx.sparse_decode_step(torch.tensor([tok], dtype=torch.int32, device="cuda"), torch.tensor([P], dtype=torch.int32, device="cuda"),
                       0, torch.zeros(1, dtype=torch.int32, device="cuda"), lo, None, ga)
torch.cuda.synchronize()
lib = S.load()
d, H, KV, hd, F = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn_dim


def buf(which, n, dt=torch.float32):
    t = torch.zeros(n, dtype=dt, device="cuda")
    lib.sirius_debug_buffer(ctx.h, 0, which, t.data_ptr(), n * t.element_size())
    return t.double().cpu().numpy()


f64 = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
resA, resB, dA = buf(0, d), buf(1, d), buf(2, d)
qkv, ob = buf(4, (H + 2 * KV) * hd), buf(5, H * hd)
Kc = buf(7, KV * MS * hd, torch.bfloat16).reshape(KV, MS, hd)
Vc = buf(8, KV * MS * hd, torch.bfloat16).reshape(KV, MS, hd)
E = lambda a, b: f"max abs {np.abs(a - b).max():.3e} (scale {np.abs(b).max():.2e})"
x0 = f64(wh["embed"][tok])
print("resA vs embed:", E(resA, x0))
h = x0 / np.sqrt(np.mean(x0 ** 2) + cfg.rms_eps) * f64(wh["layers.0.attn_norm"])
qkv_ref = f64(wh["layers.0.w_qkv"]) @ h
print("qkv (GEMV):", E(qkv, qkv_ref))
half = hd // 2
inv = cfg.rope_theta ** (-2.0 * np.arange(half) / hd)
ang = P * inv
c, s = np.cos(ang).astype(np.float32).astype(np.float64), np.sin(ang).astype(np.float32).astype(np.float64)
def rope(v):
    a, b = v[:half], v[half:]
    return np.concatenate([a * c - b * s, b * c + a * s])
q = np.stack([rope(qkv[i * hd:(i + 1) * hd]) for i in range(H)])
def attn(K, V):
    o = np.zeros((H, hd))
    for hh in range(H):
        kh = hh // (H // KV)
        sc = K[kh, :P + 1] @ q[hh] / np.sqrt(hd)
        p = np.exp(sc - sc.max()); p /= p.sum()
        o[hh] = p @ V[kh, :P + 1]
    return o.reshape(-1)
o_gc = attn(Kc, Vc)
print("attention vs fp64 on the GPU's cache:", E(ob, o_gc))
ko, vo = om.read_cache(0, P + 1)
o_oc = attn(ko.transpose(1, 0, 2), vo.transpose(1, 0, 2))
print("fp64 attention: GPU cache vs oracle cache:", E(o_gc, o_oc), " K/V elements differing:",
      int((Kc[:, :P + 1] != ko.transpose(1, 0, 2)).sum()), int((Vc[:, :P + 1] != vo.transpose(1, 0, 2)).sum()))
dA_ref = f64(wh["layers.0.w_o"]) @ ob
print("O-proj (GEMV):", E(dA, dA_ref))
print("resB vs resA + dA:", E(resB, resA + dA))
h2 = resB / np.sqrt(np.mean(resB ** 2) + cfg.rms_eps) * f64(wh["layers.0.ffn_norm"])
g = f64(wh["layers.0.w_gate"]) @ h2
a = g / (1 + np.exp(-g))
a_gpu = ga.double().cpu().numpy()[0, 0]
print("gate a (FFN kernel) vs fp64 on the GPU's resB:", E(a_gpu, a))
print("gate a: GPU vs oracle:", E(a_gpu, ref.gate[0]), " fp64-on-GPU-resB vs oracle:", E(a, ref.gate[0]))
