"""Exploration only (not product, not a test): AAL of the Sirius loop at the Llama-3-8B shape for
candidate synthetic-weight recipes.  Weights from torch RNG here; the chosen recipe is then
implemented in synth/ (both generators)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2409_03856_b200 import sirius as S, driver

cfg = synth.LLAMA3_8B
L, d, F, V = cfg.n_layers, cfg.d_model, cfg.ffn_dim, cfg.vocab
g = torch.Generator(device="cuda").manual_seed(0)

def randn(*shape, std=1.0):
    return (torch.randn(*shape, device="cuda", generator=g) * std).to(torch.bfloat16)

def make(gate_gain=None, down_gain=1.0, head_gain=5.0, up_same=True):
    w = {"embed": randn(V, d), "final_norm": torch.ones(d, device="cuda", dtype=torch.bfloat16),
         "lm_head": randn(V, d, std=head_gain / d ** 0.5)}
    for l in range(L):
        gg = gate_gain() if gate_gain else torch.ones(F, device="cuda")
        w[f"layers.{l}.attn_norm"] = torch.ones(d, device="cuda", dtype=torch.bfloat16)
        w[f"layers.{l}.ffn_norm"] = torch.ones(d, device="cuda", dtype=torch.bfloat16)
        w[f"layers.{l}.w_qkv"] = randn(cfg.qkv_rows, d, std=1 / d ** 0.5)
        w[f"layers.{l}.w_o"] = randn(d, d, std=1 / d ** 0.5)
        w[f"layers.{l}.w_gate"] = (torch.randn(F, d, device="cuda", generator=g) / d ** 0.5 * gg[:, None]).to(torch.bfloat16)
        ug = gg if up_same else torch.ones(F, device="cuda")
        w[f"layers.{l}.w_up"] = (torch.randn(F, d, device="cuda", generator=g) / d ** 0.5 * ug[:, None]).to(torch.bfloat16)
        w[f"layers.{l}.w_down"] = randn(F, d, std=down_gain / F ** 0.5)
    return w

def calibrate(w, rho=0.5):
    ctx = S.Sirius(cfg, w, [0.0] * L, batch=1, max_seq=128, max_gamma=16)
    toks = torch.tensor(synth.calib_prompt(cfg, 0, 24), dtype=torch.int32, device="cuda")
    ga = torch.zeros((1, L, F), device="cuda"); acts = []
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for i in range(24):
        ctx.sparse_decode_step(toks[i:i + 1], torch.tensor([i], dtype=torch.int32, device="cuda"), S.SIRIUS_DENSE, out, None, None, ga)
        acts.append(ga.abs().clone())
    a = torch.stack(acts)[:, 0]  # [P, L, F]
    thr = [float(torch.quantile(a[8:, l].flatten().float()[:1 << 20], 1 - rho)) for l in range(L)]
    del ctx
    return thr

def aal(w, thr, r=0.1, kernels=10):
    ctx = S.Sirius(cfg, w, thr, batch=1, max_seq=512, max_gamma=16)
    drv = driver.Driver(ctx)
    drv.begin([synth.eval_prompt(cfg, 0, 64)])
    adv = [drv.step(16, r) for _ in range(kernels)]
    drv.flush()
    del ctx
    return float(np.mean(adv)), adv

def lognormal(s):
    return lambda: torch.exp(torch.randn(F, device="cuda", generator=g) * s)

def mixture(p, big):
    return lambda: torch.where(torch.rand(F, device="cuda", generator=g) < p, torch.full((F,), big, device="cuda"), torch.ones(F, device="cuda"))

cands = {}
for hg in (5.0, 10.0):
    for name, gg, same in (("gate_up_ln1.0", lognormal(1.0), True), ("gate_up_ln1.25", lognormal(1.25), True),
                           ("gate_up_ln1.5", lognormal(1.5), True), ("gate_only_ln1.5", lognormal(1.5), False),
                           ("gate_only_ln2.0", lognormal(2.0), False)):
        cands[f"{name}_head{hg:g}"] = dict(gate_gain=gg, up_same=same, head_gain=hg)
res = {}
for name, kw in cands.items():
    t = time.time()
    w = make(**kw)
    thr = calibrate(w)
    m, adv = aal(w, thr, kernels=16)
    m3, _ = aal(w, thr, r=0.3, kernels=12)
    m5, _ = aal(w, thr, r=0.5, kernels=12)
    res[name] = dict(aal_r0_1=m, aal_r0_3=m3, aal_r0_5=m5, thr_mean=float(np.mean(thr)))
    print(name, json.dumps(res[name]), f"{time.time()-t:.1f}s", flush=True)
    del w
    torch.cuda.empty_cache()
