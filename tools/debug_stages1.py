"""Stage-isolated check of one dense decode step (last layer) against numpy, using the GPU's own
stage inputs (diagnostic tool)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S

cfg = synth.TINY.with_layers(1)
wh = synth.host_weights(cfg); wd = sg.device_weights(cfg)
thr = synth.layer_thresholds(cfg, 0.5)
c = S.Sirius(cfg, wd, thr, batch=1, max_seq=64, max_gamma=16)
lib = S.load(); lib.sirius_debug_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
def buf(which, n, dt):
    t = torch.zeros(n, dtype=dt, device="cuda"); assert lib.sirius_debug_buffer(c.h, 0, which, t.data_ptr(), t.numel()*t.element_size()) == 0
    return t.float().cpu().numpy().astype(np.float64)
f64 = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
def bf(x): return torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).double().numpy()
d, H, KV, hd, F = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn_dim
toks = synth.eval_prompt(cfg, 0, 8)
half = hd // 2
inv = 500000.0 ** (-2.0 * np.arange(half) / hd)
for P in range(4):
    to = torch.zeros(1, dtype=torch.int32, device="cuda"); lo = torch.zeros((1, cfg.vocab), device="cuda")
    c.sparse_decode_step(torch.tensor([int(toks[P])], dtype=torch.int32, device="cuda"), torch.tensor([P], dtype=torch.int32, device="cuda"), S.SIRIUS_DENSE, to, lo)
    torch.cuda.synchronize()
    l = 0
    resA = buf(0, d, torch.float32); resB = buf(1, d, torch.float32); dA = buf(2, d, torch.float32); dF = buf(3, d, torch.float32)
    qkv = buf(4, (H + 2 * KV) * hd, torch.float32); ob = buf(5, H * hd, torch.bfloat16)
    kc = buf(7, 1 * KV * 64 * hd, torch.bfloat16).reshape(1, KV, 64, hd)[l]; vc = buf(8, 1 * KV * 64 * hd, torch.bfloat16).reshape(1, KV, 64, hd)[l]
    wn = f64(wh[f"layers.{l}.attn_norm"]); h = bf(resA / np.sqrt(np.mean(resA ** 2) + 1e-5) * wn)
    q_ref = f64(wh[f"layers.{l}.w_qkv"]) @ h
    print(f"P={P} qkv err", np.abs(q_ref - qkv).max(), "scale", np.abs(q_ref).max())
    cs = np.cos(P * inv).astype(np.float32).astype(np.float64); sn = np.sin(P * inv).astype(np.float32).astype(np.float64)
    def rope(v): a, b = v[:half], v[half:]; return np.concatenate([a * cs - b * sn, b * cs + a * sn])
    q = qkv[:H * hd].reshape(H, hd); k = qkv[H * hd:(H + KV) * hd].reshape(KV, hd); v = qkv[(H + KV) * hd:].reshape(KV, hd)
    kr = np.stack([bf(rope(k[j])) for j in range(KV)]); vr = bf(v)
    print("   cache k[pos] err", np.abs(kc[:, P] - kr).max(), "v", np.abs(vc[:, P] - vr).max())
    o = np.zeros((H, hd))
    for hh in range(H):
        j = hh // (H // KV); qq = bf(rope(q[hh]))
        s = kc[j, :P + 1] @ qq / np.sqrt(hd); p = np.exp(s - s.max()); p /= p.sum(); o[hh] = bf(p @ vc[j, :P + 1])
    print("   attn out err", np.abs(o.reshape(-1) - ob).max(), "ulp-ish", np.abs(o).max() / 256)
    dA_ref = f64(wh[f"layers.{l}.w_o"]) @ ob
    print("   dA err", np.abs(dA_ref - dA).max(), "resB err", np.abs(resB - (resA + dA)).max())
    h2 = bf(resB / np.sqrt(np.mean(resB ** 2) + 1e-5) * f64(wh[f"layers.{l}.ffn_norm"]))
    g = f64(wh[f"layers.{l}.w_gate"]) @ h2; a = g / (1 + np.exp(-g)); u = f64(wh[f"layers.{l}.w_up"]) @ h2
    m = bf(a * u); dF_ref = f64(wh[f"layers.{l}.w_down"]).T @ m
    print("   dF err", np.abs(dF_ref - dF).max(), "scale", np.abs(dF_ref).max())
    x = resB + dF; hf = bf(x / np.sqrt(np.mean(x ** 2) + 1e-5) * f64(wh["final_norm"]))
    lref = f64(wh["lm_head"]) @ hf
    print("   logits err", np.abs(lref - lo.cpu().numpy()[0]).max())
from oracle import sirius_oracle as so
om = so.OracleModel(cfg, wh, max_seq=64)
c2 = S.Sirius(cfg, wd, thr, batch=1, max_seq=64, max_gamma=16)
for P in range(4):
    to = torch.zeros(1, dtype=torch.int32, device="cuda"); lo = torch.zeros((1, cfg.vocab), device="cuda")
    c2.sparse_decode_step(torch.tensor([int(toks[P])], dtype=torch.int32, device="cuda"), torch.tensor([P], dtype=torch.int32, device="cuda"), S.SIRIUS_DENSE, to, lo)
    torch.cuda.synchronize()
    r = om.decode(int(toks[P]), P, False).logits
    print("1-layer oracle vs gpu P", P, np.abs(r - lo.cpu().numpy()[0]).max())
