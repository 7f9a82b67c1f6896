"""BASELINE.json configs[4]: density x gamma x acceptance-threshold sweep on the Llama-3-8B shape
(1 B200, batch 1, 900-token prompt).  Per setting: Sirius ms/token (CUDA events over K kernels,
includes the per-kernel host round trip), AAL, correction rate (= rejected kernels / committed
tokens, PAPER.md:30 / :216), measured CATS density, effective density (Eq. 3, PAPER.md:84-87:
((n_period - 1) I + 1) / n_AAL with I = the measured global density of the sparse model).

    python tools/sweep.py [--rho 0.3,0.4,0.5,0.6,0.7] [--gamma 4,8,16,32] [--r 0.01,0.03,0.1,0.2,0.3]
                          [--kernels 32] [--out profiles/sweep_r02.csv]

Every cell starts a fresh session (dense prefill of the same prompt), runs one untimed kernel (graph
capture) and K timed kernels; AAL is reported with its standard error over the K kernels.  The
speculative-decoding baseline of the same gamma (greedy-match acceptance, EXACT_ARGMAX: a draft is
kept iff it equals the full model's argmax) is the row with r = "sd".  The
0-based draft index of every rejection is written to <out>.rejections.csv.
SM clocks are sampled with nvidia-smi during the sweep.
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
    ap.add_argument("--kernels", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=900)
    ap.add_argument("--out", default="profiles/sweep_r02.csv")
    ap.add_argument("--no-sd", action="store_true")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.model]
    w = sg.device_weights(cfg)
    prompt = synth.eval_prompt(cfg, 0, a.prompt)
    gammas, rs = lst(a.gamma, int), lst(a.r, float) + ([] if a.no_sd else ["sd"])
    gmax = max(gammas)
    rows = []
    stream = torch.cuda.current_stream()
    # sparse global density per token: gate + up/down of active neurons over all weights
    counts = {"ffn": 3 * cfg.n_layers * cfg.ffn_dim * cfg.d_model}
    total = (cfg.n_layers * (cfg.qkv_rows * cfg.d_model + cfg.d_model * cfg.n_heads * cfg.head_dim)
             + counts["ffn"] + cfg.vocab * cfg.d_model)
    import bench
    clocks = bench.Clocks(0)
    clocks.start()
    rej_rows = []
    for rho in lst(a.rho, float):
        thr = synth.layer_thresholds(cfg, rho)
        max_seq = a.prompt + (a.kernels + 3) * gmax + 64
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
        for g in gammas:
            for r in rs:
                sd = r == "sd"
                mode = S.ACCEPT_EXACT_ARGMAX if sd else S.ACCEPT_THRESHOLD
                rv = 0.0 if sd else r
                drv.flush()
                drv.begin([prompt])  # fresh session per cell (cache rewritten from the prompt)
                drv.step(g, rv, mode)  # warm-up / graph capture of this gamma
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                committed = sum(drv.step(g, rv, mode) for _ in range(a.kernels))
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                adv = np.array([int(k.j[0]) + 1 for k in drv.log[-a.kernels:]], dtype=np.float64)
                aal = committed / a.kernels
                rejected = int(np.sum(adv < g))
                for k in drv.log[-a.kernels:]:
                    if int(k.j[0]) < g - 1:
                        rej_rows.append(dict(rho_target=rho, gamma=g, r=r, rejected_at=int(k.j[0])))
                row = dict(rho_target=rho, rho_measured=round(rho_meas, 4), gamma=g, r=r,
                           ms_per_token=round(ms / committed, 4), aal=round(aal, 3),
                           aal_stderr=round(float(adv.std(ddof=1) / np.sqrt(len(adv))) if len(adv) > 1 else 0.0, 3),
                           correction_rate=round(rejected / committed, 4),
                           effective_density=round(((g - 1) * I + 1) / aal, 4), global_density_I=round(I, 4),
                           kernels=a.kernels)
                rows.append(row)
                print(row, flush=True)
        drv.flush()
        del drv, ctx
        torch.cuda.empty_cache()
    ck = clocks.stop()
    print("clocks", ck)
    for row in rows:
        row["sm_mhz_median"] = ck["sm_mhz"]
        row["clock_reasons"] = "|".join(ck["reasons"])
    with open(a.out + ".rejections.csv", "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=["rho_target", "gamma", "r", "rejected_at"])
        wr.writeheader()
        wr.writerows(rej_rows)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        wr.writeheader()
        wr.writerows(rows)
    print("wrote", a.out, len(rows), "rows")


if __name__ == "__main__":
    main()
