"""Per-rank timing proxy of tensor-parallel decode on ONE GPU (BASELINE.json configs[2] / configs[3]):
a context holding exactly one rank's shard (tp_size = N, tp_rank = 0) with every collective skipped
(SIRIUS_DEBUG_STUB_COMM=1, include/sirius.h) — the compute a rank of an N-GPU group runs per token,
without the NVLink all-reduces (2 per layer + the head's max-reduce + the accept all-gather).  Not a
multi-GPU measurement: the all-reduce latency must be added (65 calls per 8B token,
161 per 70B token, 16 / 32 KB each at batch 1).  Outputs are rank-local partials, so r = 0 keeps the
kernel shape fixed (advance = gamma) and the Sirius number is reported per committed token at
AAL = gamma and, as a model, at the TP-1 bench's AAL.

    python tools/tp_proxy.py --model llama3-8b --tp 8 [--batch 1] [--gamma 16] [--steps 8] [--par]

--par: the fused peer all-reduce in loopback (sirius_par_enable on a stub context): the decode step's
pushes, flag stores and waits run on-chip against the rank's own buffer (every "peer" is itself), so
the proxy then includes the fused all-reduce's in-kernel cost — all but the NVLink transfer latency.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SIRIUS_DEBUG_STUB_COMM"] = "1"
import numpy as np, torch
import synth, bench
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--tp", type=int, default=8)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--gamma", type=int, default=16)
ap.add_argument("--prompt", type=int, default=900)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--rho", type=float, default=0.5)
ap.add_argument("--out", default=None)
ap.add_argument("--par", action="store_true")
a = ap.parse_args()
cfg = synth.CONFIGS[a.model]
t0 = time.time()
w = sg.device_weights(cfg, a.tp, 0)
thr = synth.layer_thresholds(cfg, a.rho)
B, g = a.batch, a.gamma
max_seq = a.prompt + (a.warmup + a.steps + 4) * g + 256
ctx = S.Sirius(cfg, w, thr, batch=B, max_seq=max_seq, max_gamma=g, tp_size=a.tp, tp_rank=0, nccl_comm=1)
if a.par:
    ctx.sirius_par_enable(None)
drv = driver.Driver(ctx)
prompts = [synth.eval_prompt(cfg, b, a.prompt) for b in range(B)]
drv.begin(prompts)
setup = time.time() - t0
st = torch.cuda.current_stream()
clk = bench.Clocks(0)
clk.start()
for _ in range(a.warmup):
    drv.step(g, 0.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(a.steps):
    drv.step(g, 0.0)
e1.record(st)
torch.cuda.synchronize()
t_kernel = e0.elapsed_time(e1) / a.steps
base = {}
T0 = [t + 8 for t in drv.T]
for name, dense in (("dense", True), ("cs_only", False)):
    drv.greedy_run(drv.pending, T0, g, dense)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(st)
    drv.greedy_run(drv.pending, T0, 64, dense)
    f1.record(st)
    torch.cuda.synchronize()
    base[name] = f0.elapsed_time(f1) / 64
# per kernel class: device us per CS decode step (CUDA events around every launch, graphs on)
ctx.profile(True)
drv.greedy_run(drv.pending, T0, 16, False)
torch.cuda.synchronize()
prof = {k: v[0] * 1e3 / 16 for k, v in ctx.profile_read().items() if v[1]}
ctx.profile(False)
ctx.profile(True)  # the correction kernel (verify forward + accept), per call
for _ in range(3):
    drv.step(g, 0.0)
torch.cuda.synchronize()
pr = ctx.profile_read()
verify_us = pr["correct_kernel"][0] * 1e3 / max(1, pr["correct_kernel"][1])
ctx.profile(False)
ck = clk.stop()
tp_per_rank = dict(ffn=cfg.ffn_dim // a.tp, heads=cfg.n_heads // a.tp, kv_heads=cfg.n_kv_heads // a.tp,
                   vocab=cfg.vocab // a.tp)
dense_bytes = bench.step_bytes(cfg, a.tp, drv.T[0], None, B)
what = (f"{a.model} TP{a.tp} per-rank proxy on 1 B200, decode all-reduces fused + looped back on-chip "
        "(verify collectives skipped)") if a.par else f"{a.model} TP{a.tp} per-rank compute proxy on 1 B200 (collectives skipped)"
res = {"what": what, "fused_peer_allreduce_loopback": a.par, "batch": B,
       "gamma": g, "prompt": a.prompt, "shard": tp_per_rank,
       "dense_ms_per_token": base["dense"], "cs_only_ms_per_token": base["cs_only"],
       "sirius_ms_per_kernel": t_kernel, "sirius_ms_per_token_at_aal_gamma": t_kernel / g,
       "dense_hbm_gbs": dense_bytes / (base["dense"] / 1e3) / 1e9,
       "dense_bytes_per_rank": dense_bytes,
       "allreduces_per_token": 2 * cfg.n_layers + 1,
       "note": ("add the NVLink transfer latency of each fused push (not measured: one GPU)" if a.par else
                "add the NVLink all-reduce latency per call (not measured: one GPU)"),
       "cs_step_device_us_by_kernel_class": prof,
       "correct_kernel_device_us": verify_us,
       "clocks": ck, "setup_s": setup}
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
