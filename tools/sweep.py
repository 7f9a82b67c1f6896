"""BASELINE.json configs[4]: density x gamma x acceptance-threshold sweep on the Llama-3-8B shape
(1 B200, batch 1, 900-token prompt).  Per setting: Sirius ms/token (CUDA events over K kernels,
includes the per-kernel host round trip), AAL, correction rate (= rejected kernels / committed
tokens, PAPER.md:30 / :216), measured CATS density, effective density (Eq. 3, PAPER.md:84-87:
((n_period - 1) I + 1) / n_AAL with I = the measured global density of the sparse model).

    python tools/sweep.py [--rho 0.3,0.4,0.5,0.6,0.7] [--gamma 4,8,16,32] [--r 0.01,0.03,0.1,0.2,0.3]
                          [--kernels 6] [--out profiles/sweep_r01.csv]
"""
import argparse
import csv
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2409_03856_b200 import driver, sirius as S  # noqa: E402
from synth import gpu as sg  # noqa: E402


def lst(s, f):
    return [f(x) for x in s.split(",")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--rho", default="0.3,0.4,0.5,0.6,0.7")
    ap.add_argument("--gamma", default="4,8,16,32")
    ap.add_argument("--r", default="0.01,0.03,0.1,0.2,0.3")
    ap.add_argument("--kernels", type=int, default=6)
    ap.add_argument("--prompt", type=int, default=900)
    ap.add_argument("--out", default="profiles/sweep_r01.csv")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.model]
    w = sg.device_weights(cfg)
    prompt = synth.eval_prompt(cfg, 0, a.prompt)
    gammas, rs = lst(a.gamma, int), lst(a.r, float)
    gmax = max(gammas)
    rows = []
    stream = torch.cuda.current_stream()
    # sparse global density per token: gate + up/down of active neurons over all weights
    counts = {"ffn": 3 * cfg.n_layers * cfg.ffn_dim * cfg.d_model}
    total = (cfg.n_layers * (cfg.qkv_rows * cfg.d_model + cfg.d_model * cfg.n_heads * cfg.head_dim)
             + counts["ffn"] + cfg.vocab * cfg.d_model)
    for rho in lst(a.rho, float):
        thr = synth.layer_thresholds(cfg, rho)
        max_seq = a.prompt + (len(rs) * (a.kernels + 2) + 4) * gmax + 64
        ctx = S.Sirius(cfg, w, thr, batch=1, max_seq=max_seq, max_gamma=gmax)
        drv = driver.Driver(ctx)
        drv.begin([prompt])
        # measured CATS density of this threshold set (8 sparse steps)
        na = torch.zeros((1, cfg.n_layers), dtype=torch.int32, device="cuda")
        tok = torch.tensor([drv.pending[0]], dtype=torch.int32, device="cuda")
        out = torch.zeros(1, dtype=torch.int32, device="cuda")
        dens = []
        for i in range(8):
            ctx.sparse_decode_step(tok, torch.tensor([a.prompt + i], dtype=torch.int32, device="cuda"), 0, out, None, na)
            dens.append(na.cpu().numpy()[0] / cfg.ffn_dim)
        rho_meas = float(np.mean(dens))
        # global density I of the sparse model (gate dense, up/down scaled by rho_meas)
        sparse_params = total - counts["ffn"] + cfg.n_layers * cfg.ffn_dim * cfg.d_model * (1 + 2 * rho_meas)
        I = sparse_params / total
        drv.begin([prompt])  # fresh session (cache rewritten from the prompt)
        for g in gammas:
            for r in rs:
                drv.step(g, r)  # warm-up / graph capture of this gamma
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                committed = sum(drv.step(g, r) for _ in range(a.kernels))
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                adv = [int(k.j[0]) + 1 for k in drv.log[-a.kernels:]]
                aal = committed / a.kernels
                rejected = sum(1 for x in adv if x < g)
                row = dict(rho_target=rho, rho_measured=round(rho_meas, 4), gamma=g, r=r,
                           ms_per_token=round(ms / committed, 4), aal=round(aal, 3),
                           correction_rate=round(rejected / committed, 4),
                           effective_density=round(((g - 1) * I + 1) / aal, 4), global_density_I=round(I, 4),
                           kernels=a.kernels)
                rows.append(row)
                print(row, flush=True)
                if drv.T[0] + (a.kernels + 2) * gmax >= max_seq:
                    drv.flush()
                    drv.begin([prompt])
        drv.flush()
        del drv, ctx
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        wr.writeheader()
        wr.writerows(rows)
    print("wrote", a.out, len(rows), "rows")


if __name__ == "__main__":
    main()
