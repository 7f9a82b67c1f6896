"""Full-model verification latency vs kernel size (the B200 analogue of PAPER.md Table 10, P:643-676:
"length 64 is only 1.1 ms longer than length 1").  Llama-3-8B shape,
batch 1, 900-token context; correct_kernel timed with CUDA events (graph replays, median of 7).

    python tools/verify_gamma.py [--out profiles/verify_gamma_r01.csv]
"""
import argparse
import csv
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2409_03856_b200 import sirius as S  # noqa: E402
from synth import gpu as sg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/verify_gamma_r01.csv")
    ap.add_argument("--prompt", type=int, default=900)
    a = ap.parse_args()
    cfg = synth.CONFIGS["llama3-8b"]
    gammas = [1, 2, 4, 8, 16, 32, 64]
    ctx = S.Sirius(cfg, sg.device_weights(cfg), synth.layer_thresholds(cfg, 0.5), batch=1,
                   max_seq=a.prompt + 128, max_gamma=max(gammas))
    prompt = synth.eval_prompt(cfg, 0, a.prompt)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(torch.tensor(prompt, dtype=torch.int32, device="cuda"), [a.prompt], f)
    start = torch.tensor([a.prompt], dtype=torch.int32, device="cuda")
    na = torch.zeros(1, dtype=torch.int32, device="cuda")
    nx = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    rows = []
    for g in gammas:
        kt = f.repeat(g).view(1, g).contiguous()
        times = []
        for it in range(9):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.correct_kernel(kt, start, g, 0.1, 0, na, nx)
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        rows.append({"gamma": g, "rows": g, "verify_ms": round(ms, 4), "ms_per_row": round(ms / g, 4)})
        print(rows[-1], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)


if __name__ == "__main__":
    main()
