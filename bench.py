#!/usr/bin/env python3
"""bench.py — Sirius decode on Llama-3-8B-shaped random weights (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sirius|reference]

A *step* is one pass of the whole hot path: one Sirius correction kernel
= gamma-1 CATS-sparse decode steps (S1-S7) + the full-model verification of the kernel (S8) + the
likelihood accept/reject and interleave (S9) + the KV rewrite of the committed span (S10).
Metric (BASELINE.json): decode ms/token & HBM GB/s, Sirius vs dense vs CS-only.  `value` is the
Sirius decode latency per committed token (lower is better); dense and CS-only latencies of the
same library are reported beside it.  N > 1: tensor parallel over N GPUs (NCCL all-reduce per
layer), every rank runs the same loop; timing = max over ranks.
--impl reference: the CPU oracle (oracle/) timed on the host cores on a bounded sample of the same
workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

WORKLOAD = "llama3-8b-shape random-init bf16, batch 1, prompt 900, CATS 50% FFN density, gamma 16, r 0.1"
METRIC = "decode ms/token (Sirius; dense and CS-only beside it), Llama-3-8B shape"


def bench_config(a, world):
    """The workload description shared by both arms (BASELINE.json configs[1] by default)."""
    B = a.batch
    return {"workload": WORKLOAD if B == 1 else WORKLOAD.replace("batch 1", f"batch {B}"), "model": a.model,
            "batch": B, "prompt": a.prompt, "gamma": a.gamma, "r": a.r, "rho_target": a.rho,
            "parallelism": f"tp{world}",
            "l2": "weights (15 GB) >> 126 MB L2: every step streams from HBM, no flush needed"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sirius", choices=["sirius", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--prompt", type=int, default=900)
    ap.add_argument("--gamma", type=int, default=16)
    ap.add_argument("--r", type=float, default=0.1)
    ap.add_argument("--r-alt", type=float, default=0.3,
                    help="second acceptance threshold timed beside the main one (an operating point with rejections)")
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--batch", type=int, default=1, help="sequences decoded together (1, 2, 4, 8)")
    ap.add_argument("--baseline-tokens", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tree-width", type=int, default=4, help="tree kernels timed at r_alt (0: skip)")
    ap.add_argument("--topk-keep", type=float, default=0.5, help="top-k FSparse rows (0: skip)")
    ap.add_argument("--csparse-keep", type=float, default=0.5,
                    help="CSparse (Griffin-style) keep fraction for the csparse rows (0: skip)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# ---------------------------------------------------------------- algorithmic bytes
def step_bytes(cfg, tp, ctx_len, rho_layers=None, batch=1):
    """Bytes the method must move for one decode step of `batch` sequences per rank: weights (dense,
    or CATS-sparse FFN with rho_layers = the active fraction per layer, the union over the batch
    for batch > 1) read once + each sequence's KV-cache read of ctx_len positions + the head."""
    d, F, L, hd = cfg.d_model, cfg.ffn_dim // tp, cfg.n_layers, cfg.head_dim
    qkv = cfg.qkv_rows // tp * d * 2
    wo = d * (cfg.n_heads // tp * hd) * 2
    gate = F * d * 2
    kv = batch * 2 * (cfg.n_kv_heads // tp) * hd * 2 * ctx_len
    tot = 0.0
    for l in range(L):
        rho = 1.0 if rho_layers is None else float(rho_layers[l])
        tot += qkv + wo + gate + 2 * rho * F * d * 2 + kv
    tot += cfg.vocab // tp * d * 2
    return tot


def verify_bytes(cfg, tp, T, gamma, batch=1):
    d, F, L, hd = cfg.d_model, cfg.ffn_dim // tp, cfg.n_layers, cfg.head_dim
    w = L * (cfg.qkv_rows // tp * d + d * cfg.n_heads // tp * hd + 3 * F * d) * 2 + cfg.vocab // tp * d * 2
    kvrow = 2 * (cfg.n_kv_heads // tp) * hd * 2 * L
    return w + batch * (T * kvrow + gamma * kvrow + gamma * cfg.vocab // tp * 4)


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self, index=0):
        self.samples, self.proc, self.index = [], None, index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 7 for i in range(4)
                          if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------- CPU oracle baseline
class OracleSample:
    """The oracle as it stands, on a bounded sample of the workload: one Sirius kernel (gamma-1
    CATS-sparse rows + gamma dense verify rows) of the 2-layer truncation of the model, plus head-only
    rows; the per-row cost is scaled to the full depth, t(L) = t_head + L/2 * (t(2 layers) - t_head).
    Weights are generated once (outside the timed samples)."""

    def __init__(self, cfg_full, gamma, rho, prompt_len=4):
        from oracle import sirius_oracle as so
        self.so, self.cfg, self.gamma, self.P = so, cfg_full, gamma, prompt_len
        cfg2 = cfg_full.with_layers(2)
        w = synth.host_weights(cfg2)
        self.thr = synth.layer_thresholds(cfg2, rho)
        self.m = so.OracleModel(cfg2, w, max_seq=prompt_len + 2 * gamma + 4, max_gamma=gamma)
        self.m0 = so.OracleModel(cfg_full.with_layers(0), {k: v for k, v in w.items() if not k.startswith("layers")},
                                 max_seq=8)
        self.prompt = synth.eval_prompt(cfg2, 0, prompt_len)
        self.threads = self.m.threads

    def run(self):
        """One sample; returns the per-row costs at full depth and the sample's own wall time."""
        so, g, P = self.so, self.gamma, self.P
        w0 = time.perf_counter()
        self.m.prefill(self.prompt)
        tok = 7
        t0 = time.perf_counter()
        drafts = [tok]
        for i in range(g - 1):
            row = self.m.decode(drafts[-1], P + i, True, self.thr)
            drafts.append(so.argmax_lowest(row.logits))
        t_sparse = (time.perf_counter() - t0) / (g - 1)
        t0 = time.perf_counter()
        self.m.verify(drafts, P)
        t_dense = (time.perf_counter() - t0) / g
        t0 = time.perf_counter()
        for _ in range(3):
            self.m0.forward_row(5, 0)
        t_head = (time.perf_counter() - t0) / 3
        half = self.cfg.n_layers / 2.0
        return dict(row_sparse_s=t_head + half * (t_sparse - t_head), row_dense_s=t_head + half * (t_dense - t_head),
                    sample_s=time.perf_counter() - w0)

    def ms_per_token(self, s, advance):
        """Sirius ms per committed token at full depth: (gamma-1 sparse rows + gamma verify rows) / advance."""
        return ((self.gamma - 1) * s["row_sparse_s"] + self.gamma * s["row_dense_s"]) / advance * 1e3

    def describe(self, advance_note):
        return (f"per sample: one gamma={self.gamma} Sirius kernel ({self.gamma - 1} CATS-sparse rows + {self.gamma} "
                f"dense verify rows) of the 2-layer truncation of the {self.cfg.name} shape + head-only rows, oracle "
                f"timed as it stands and scaled to {self.cfg.n_layers} layers; {advance_note}")


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[a.model]
    t_start = time.perf_counter()
    osm = OracleSample(cfg, a.gamma, a.rho)
    vals, walls = [], []
    for i in range(a.warmup + a.steps):
        s = osm.run()
        if i >= a.warmup:
            vals.append(osm.ms_per_token(s, a.gamma))
            walls.append(s["sample_s"])
    v = statistics.median(vals)
    sample = osm.describe("advance taken as gamma (the GPU arm measures AAL 16.0/16 at r = 0.1); one step = one "
                          "sample, ms_per_step = its measured wall time")
    out = {"metric": METRIC, "value": v, "unit": "ms/token",
           "impl": "reference", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
           "ms_per_step": statistics.mean(walls) * 1e3,
           "higher_is_better": False, "dtype": "f64", "data": "synthetic",
           "config": bench_config(a, int(os.environ.get("WORLD_SIZE", "1"))),
           "cpu_baseline": {"value": v, "unit": "ms/token", "cores": osm.threads, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "wall_s": time.perf_counter() - t_start}
    print(json.dumps(out))


# ---------------------------------------------------------------- GPU arm
def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    from paper_2409_03856_b200 import driver, sirius as S, tp as TP
    from synth import gpu as sg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.gpus > 1 and world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} needs torchrun with {a.gpus} ranks (WORLD_SIZE={world})")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    cfg = synth.CONFIGS[a.model]
    tp = world
    t_setup = time.perf_counter()
    weights = sg.device_weights(cfg, tp, rank)
    thr = synth.layer_thresholds(cfg, a.rho)
    comm = None
    if tp > 1:
        comm = TP.nccl_bootstrap(S.load(), tp, rank)
    n_gen_max = (a.warmup + 2 * a.steps + 2) * a.gamma + a.baseline_tokens + 64
    max_seq = a.prompt + n_gen_max + 2 * a.gamma
    B = a.batch
    ctx = S.Sirius(cfg, weights, thr, batch=B, max_seq=max_seq, max_gamma=a.gamma, tp_size=tp, tp_rank=rank,
                   nccl_comm=comm)
    drv = driver.Driver(ctx)
    prompts = [synth.eval_prompt(cfg, b, a.prompt) for b in range(B)]
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    barrier, max_over_ranks = TP.barrier, TP.max_over_ranks

    stream = torch.cuda.current_stream()
    # ---------------- Sirius: W warm-up kernels, then K timed kernels
    drv.begin(prompts)
    for _ in range(a.warmup):
        drv.step(a.gamma, a.r)
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches()
    h2d0, d2h0 = drv.h2d_bytes, drv.d2h_bytes
    wall0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(a.steps):
        drv.step(a.gamma, a.r)
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    barrier()
    ck = clocks.stop()
    launches = ctx.launches() - l0
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    wall_ms = max_over_ranks(wall * 1e3)
    h2d = (drv.h2d_bytes - h2d0) / a.steps
    d2h = (drv.d2h_bytes - d2h0) / a.steps
    timed = drv.log[a.warmup:a.warmup + a.steps]
    advances = [[int(x) + 1 for x in k.j] for k in timed]  # [kernel][sequence]
    committed_total = sum(sum(v) for v in advances)
    committed = committed_total / B  # per sequence
    aal = committed / a.steps
    sirius_ms_tok = t_ms / committed  # per-sequence latency per committed token
    # ---------------- roofline pass: per-kernel CUDA events over K more kernels
    ctx.profile(True)
    for _ in range(a.steps):
        drv.step(a.gamma, a.r)
    prof = ctx.profile_read()
    ctx.profile(False)
    T_now = drv.T[0]
    drv.flush()
    # measured CATS density per layer (sparse steps with gate-activation export): per sequence and
    # the union over the batch (the rows a batched step must load, reading D19)
    L, Fr_ = cfg.n_layers, cfg.ffn_dim // tp
    tok = torch.tensor(drv.pending, dtype=torch.int32, device="cuda")
    tok2 = torch.zeros(B, dtype=torch.int32, device="cuda")
    ga = torch.zeros((B, L, Fr_), dtype=torch.float32, device="cuda")
    thr_np = np.asarray(thr, dtype=np.float32)[None, :, None]
    dens, union = [], []
    for i in range(8):
        p = torch.tensor([t + i for t in drv.T], dtype=torch.int32, device="cuda")
        ctx.sparse_decode_step(tok, p, 0, tok2, None, None, ga)
        tok.copy_(tok2)
        act = np.abs(ga.cpu().numpy()) >= thr_np  # [B, L, F]
        dens.append(act.mean(axis=2).mean(axis=0))
        union.append(act.any(axis=0).mean(axis=1))
    rho_layers = np.mean(np.array(dens), axis=0)
    rho_union = np.mean(np.array(union), axis=0)
    # ---------------- dense and CS-only baselines (same library, same context)
    n_b = a.baseline_tokens
    T0 = [t + 8 for t in drv.T]
    base = {}
    for name, dense in (("dense", True), ("cs_only", False)):
        drv.greedy_run(drv.pending, T0, a.gamma, dense)  # warm-up: captures the chunk's graphs
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        drv.greedy_run(drv.pending, T0, n_b, dense)
        e1.record(stream)
        torch.cuda.synchronize()
        base[name] = max_over_ranks(e0.elapsed_time(e1)) / n_b
    # ---------------- a second operating point where the correction fires (rollback + interleave inside
    # the timed region): fresh session, W warm-up kernels, K timed kernels at r = r_alt
    alt = None
    if a.r_alt is not None and a.r_alt != a.r:
        drv.begin(prompts)
        for _ in range(a.warmup):
            drv.step(a.gamma, a.r_alt)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            drv.step(a.gamma, a.r_alt)
        e1.record(stream)
        torch.cuda.synchronize()
        t_alt = max_over_ranks(e0.elapsed_time(e1))
        tl = drv.log[a.warmup:a.warmup + a.steps]
        adv_alt = [[int(x) + 1 for x in k.j] for k in tl]
        c_alt = sum(sum(v) for v in adv_alt) / B
        alt = {"r": a.r_alt, "ms_per_token": t_alt / c_alt, "aal": c_alt / a.steps,
               "advances": adv_alt if B > 1 else [v[0] for v in adv_alt],
               "rejected_kernels": int(sum(1 for v in adv_alt for x in v if x < a.gamma)),
               "rejection_positions": [int(k.j[b]) for k in tl for b in range(B) if int(k.j[b]) < a.gamma - 1],
               "vs_dense": (t_alt / c_alt) / base["dense"]}
        drv.flush()
    # ---------------- tree building + tree verification at r_alt: the tree's AAL against
    # the chain's at the same threshold, and its cost per kernel
    tree = None
    if a.tree_width > 0 and B == 1 and tp == 1 and 1 + (a.gamma - 1) * a.tree_width <= 64 and alt is not None:
        ctx_t = S.Sirius(cfg, weights, thr, batch=1, max_seq=max_seq, max_gamma=64)
        dt = driver.Driver(ctx_t)
        dt.begin(prompts)
        for _ in range(a.warmup):
            dt.step_tree(a.gamma, a.r_alt, a.tree_width)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            dt.step_tree(a.gamma, a.r_alt, a.tree_width)
        e1.record(stream)
        torch.cuda.synchronize()
        t_tree = max_over_ranks(e0.elapsed_time(e1))
        adv_t = [int(k.j[0]) + 1 for k in dt.log[a.warmup:a.warmup + a.steps]]
        dt.flush()
        tree = {"width": a.tree_width, "branch": 3, "r": a.r_alt, "rows_verified": 1 + (a.gamma - 1) * a.tree_width,
                "aal": sum(adv_t) / a.steps, "aal_chain_same_r": alt["aal"], "ms_per_kernel": t_tree / a.steps,
                "ms_per_token": t_tree / sum(adv_t),
                "note": "tree drafting runs W rows per step through the verify-row machinery (tcgen05 GEMMs over "
                        "all FFN rows, ancestor-masked attention): ~a verify pass per step"}
        del dt, ctx_t
        torch.cuda.empty_cache()
    # ---------------- top-k FSparse (the paper's own FSparse, PAPER.md:121 footnote): Sirius and sparse-only
    tk = None
    if a.topk_keep > 0 and tp == 1 and B <= 4:
        ctx.sirius_topk_enable(a.topk_keep)
        dk = driver.Driver(ctx, topk=True)
        dk.begin(prompts)
        for _ in range(a.warmup):
            dk.step(a.gamma, a.r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            dk.step(a.gamma, a.r)
        e1.record(stream)
        torch.cuda.synchronize()
        t_k = max_over_ranks(e0.elapsed_time(e1))
        adv_k = [int(k.j[0]) + 1 for k in dk.log[a.warmup:a.warmup + a.steps]]
        dk.flush()
        Tk = [t + 8 for t in dk.T]
        dk.greedy_run(dk.pending, Tk, a.gamma, False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dk.greedy_run(dk.pending, Tk, a.baseline_tokens, False)
        e1.record(stream)
        torch.cuda.synchronize()
        tk = {"keep": a.topk_keep, "sirius_ms_per_token": t_k / sum(adv_k), "aal": sum(adv_k) / a.steps,
              "sparse_only_ms_per_token": max_over_ranks(e0.elapsed_time(e1)) / a.baseline_tokens}
        ctx.sirius_topk_enable(0.0)
    # ---------------- CSparse (Griffin-style, the sparse model of the paper's latency tables):
    # the same context with the prompt's fixed neuron set; Sirius over the CSparse draft model, and
    # CSparse-only greedy decode
    csp = None
    if a.csparse_keep > 0 and B == 1:
        ctx.sirius_csparse_enable(a.csparse_keep)
        dcs = driver.Driver(ctx, csparse=True)
        dcs.begin(prompts)
        for _ in range(a.warmup):
            dcs.step(a.gamma, a.r)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            dcs.step(a.gamma, a.r)
        e1.record(stream)
        torch.cuda.synchronize()
        t_cs_sir = max_over_ranks(e0.elapsed_time(e1))
        adv_cs = [int(k.j[0]) + 1 for k in dcs.log[a.warmup:a.warmup + a.steps]]
        dcs.flush()
        Tc = [t + 8 for t in dcs.T]
        dcs.greedy_run(dcs.pending, Tc, a.gamma, False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dcs.greedy_run(dcs.pending, Tc, a.baseline_tokens, False)
        e1.record(stream)
        torch.cuda.synchronize()
        t_cs_only = max_over_ranks(e0.elapsed_time(e1)) / a.baseline_tokens
        kk = int(np.floor(a.csparse_keep * cfg.ffn_dim // tp + 0.5))
        cs_bytes = step_bytes(cfg, tp, dcs.T[0], None, B) - cfg.n_layers * 3 * (cfg.ffn_dim // tp - kk) * cfg.d_model * 2
        csp = {"keep": a.csparse_keep, "neurons_per_layer": kk,
               "sirius_ms_per_token": t_cs_sir / sum(adv_cs), "aal": sum(adv_cs) / a.steps,
               "cs_only_ms_per_token": t_cs_only, "cs_only_hbm_gbs": cs_bytes / (t_cs_only / 1e3) / 1e9,
               "sirius_vs_dense": (t_cs_sir / sum(adv_cs)) / base["dense"],
               "global_density": cs_bytes / step_bytes(cfg, tp, dcs.T[0], None, B)}
        ctx.sirius_csparse_enable(0.0)
    # ---------------- latency model: per committed token
    # ((gamma-1) t_CS + t_verify + t_rewrite + t_host) / AAL, the components measured above
    t_ver = prof.get("correct_kernel", (0.0, 0))
    t_rw = prof.get("kv_rewrite", (0.0, 0))
    t_verify = t_ver[0] / max(t_ver[1], 1)
    t_rewrite = t_rw[0] / max(t_rw[1], 1)
    t_step = t_ms / a.steps
    t_host = t_step - ((a.gamma - 1) * base["cs_only"] + t_verify + t_rewrite)
    kern_ms = (a.gamma - 1) * base["cs_only"] + t_verify + t_rewrite + max(t_host, 0.0)
    model = {"components_ms": {"t_cs": base["cs_only"], "t_dense": base["dense"], "t_verify": t_verify,
                               "t_rewrite": t_rewrite, "t_host_and_overlap": t_host, "kernel": kern_ms},
             "ms_per_token_at_aal": {str(x): kern_ms / x for x in range(a.gamma // 2, a.gamma + 1, 2)},
             "break_even_aal_vs_dense": kern_ms / base["dense"],
             "note": "model, labelled as such: the measured points are sirius (r) and sirius_r_alt"}
    # ---------------- roofline of the dominant kernel: the persistent decode step (TP 1), else the CATS FFN
    pk = peaks()
    d, Fr = cfg.d_model, cfg.ffn_dim // tp
    rho_mean = float(np.mean(rho_layers))
    rho_union_mean = float(np.mean(rho_union))
    traffic = None
    summ = {}
    try:
        for tag in ("r02", "r01"):  # the latest committed ncu --set full summary
            pth = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")
            if os.path.exists(pth):
                summ = json.load(open(pth))
                break
    except Exception:
        pass
    if prof.get("decode_step", (0.0, 0))[1] > 0:
        st_ms, st_n = prof["decode_step"]
        # algorithmic bytes of one CATS-sparse step at the mean context of the timed kernels
        ctx_mid = T_now - a.steps * a.gamma / 2
        st_bytes = step_bytes(cfg, tp, ctx_mid, rho_union, B)
        avg_s = st_ms / st_n / 1e3
        achieved = st_bytes / avg_s / 1e9
        try:
            traffic = summ["kernels"]["decode_step_kernel"]["dram_bytes_per_launch"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": ("decode_step_kernel (persistent CATS-sparse decode step: QKV, attention, "
                "O-proj, gate+SiLU+threshold+ballot, active up/down gathers, head+argmax)") if B < 8 else
                "batched decode step (row path: tcgen05 GEMMs with the CATS-masked SwiGLU epilogue, attention, head)",
                "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                "traffic": traffic, "algorithmic_bytes_per_launch": st_bytes, "avg_launch_us": avg_s * 1e6,
                "launches_timed": st_n,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in pk else "fallback (B200_PROFILING.md)"}
    else:
        ffn_ms, ffn_n = prof["cats_ffn"]
        ffn_bytes = Fr * d * 2 + 2 * rho_union_mean * Fr * d * 2  # dense gate + active (union) up/down rows
        ffn_avg_s = ffn_ms / max(ffn_n, 1) / 1e3
        achieved = ffn_bytes / ffn_avg_s / 1e9
        try:
            traffic = summ["cats_ffn"]["dram_bytes_per_launch"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": "ffn_kernel (CATS gate+SiLU+threshold+ballot, active up/down gathers)",
                "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                "traffic": traffic, "algorithmic_bytes_per_launch": ffn_bytes, "avg_launch_us": ffn_avg_s * 1e6,
                "launches_timed": ffn_n,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in pk else "fallback (B200_PROFILING.md)"}
    # whole-step HBM GB/s for each mode (algorithmic bytes / time)
    ctxlen = T_now
    gbs = {"dense": step_bytes(cfg, tp, ctxlen, None, B) / (base["dense"] / 1e3) / 1e9,
           "cs_only": step_bytes(cfg, tp, ctxlen, rho_union, B) / (base["cs_only"] / 1e3) / 1e9}
    kernel_bytes = ((a.gamma - 1) * step_bytes(cfg, tp, ctxlen, rho_union, B)
                    + verify_bytes(cfg, tp, ctxlen, a.gamma, B))
    gbs["sirius"] = kernel_bytes / (t_ms / a.steps / 1e3) / 1e9
    per_kernel = {k: {"ms_total": v[0], "launches": v[1]} for k, v in prof.items()}
    # ---------------- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and B == 1 and not a.no_cpu_baseline:
        osm = OracleSample(cfg, a.gamma, a.rho)
        ss = [osm.run() for _ in range(3)]
        v = statistics.median(osm.ms_per_token(x, aal) for x in ss)
        cpu = {"value": v, "unit": "ms/token", "cores": osm.threads, "kind": "oracle",
               "sample": osm.describe(f"divided by the GPU-measured AAL {aal:.2f}; median of 3 samples"),
               "row_sparse_s": statistics.median(x["row_sparse_s"] for x in ss),
               "row_dense_s": statistics.median(x["row_dense_s"] for x in ss)}
    if rank == 0:
        out = {
            "metric": METRIC,
            "value": sirius_ms_tok, "unit": "ms/token", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": t_ms / a.steps, "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": bench_config(a, world),
            "sirius": {"ms_per_token": sirius_ms_tok, "aal": aal,
                       "advances": advances if B > 1 else [v[0] for v in advances],
                       "tokens_per_s": 1e3 / sirius_ms_tok, "tokens_per_s_aggregate": B * 1e3 / sirius_ms_tok,
                       "hbm_gbs_algorithmic": gbs["sirius"]},
            "dense": {"ms_per_token": base["dense"], "tokens_per_s": 1e3 / base["dense"], "hbm_gbs": gbs["dense"],
                      "frac_of_measured_hbm": gbs["dense"] / pk["hbm_gbs"]},
            "cs_only": {"ms_per_token": base["cs_only"], "tokens_per_s": 1e3 / base["cs_only"],
                        "hbm_gbs": gbs["cs_only"], "frac_of_measured_hbm": gbs["cs_only"] / pk["hbm_gbs"],
                        "density_per_layer_mean": rho_mean, "density_union_over_batch": rho_union_mean,
                        "tokens_per_s_aggregate": B * 1e3 / base["cs_only"]},
            "sirius_vs_dense": sirius_ms_tok / base["dense"],
            "sirius_r_alt": alt,
            "csparse": csp,
            "tree": tree,
            "topk_fsparse": tk,
            "latency_model": model,
            "roofline": roof, "per_kernel_device_ms": per_kernel,
            "cpu_baseline": cpu,
            "e2e": {"value": wall_ms / committed, "unit": "ms/token", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "note": "wall clock of the same K kernels through the C ABI; per kernel the positions/pending "
                            "token go H2D from pinned host memory and the accepted count + drafted tokens come back D2H"},
            "gpu_launches": launches,
            "cuda_graphs": ctx.graphs(),
            "clocks": ck,
            "setup_s": setup_s,
        }
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
