"""Steady-state timing of the tcgen05 verify GEMM alone (sirius_debug_gemm), rotating over enough
distinct weight copies that every launch streams from HBM.  Shapes: the Llama-3-8B verify GEMMs
(QKV, O, gate+up dual, down) at M token rows.  Debug tool, not a bench value."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_03856_b200 import sirius as S

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, nargs="+", default=[16])
ap.add_argument("--terms", type=int, nargs="+", default=[3])
ap.add_argument("--reps", type=int, default=16)
a = ap.parse_args()
lib = S.load()
shapes = {"qkv": (6144, 4096, False), "o": (4096, 4096, False), "gate+up": (14336, 4096, True), "down": (4096, 14336, False)}
for name, (N, K, dual) in shapes.items():
    ncopy = max(2, int(400e6 // (N * K * 2 * (2 if dual else 1))) + 1)
    W = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.02 for _ in range(ncopy)]
    W2 = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.02 for _ in range(ncopy)] if dual else None
    for M in a.m:
        for nt in a.terms:
            X = (torch.randn(nt, 256, K, device="cuda") * 0.1).to(torch.bfloat16)
            out = torch.zeros(3 * M * N if dual else M * N, device="cuda", dtype=torch.bfloat16 if dual else torch.float32)
            ts = []
            for r in range(a.reps + 2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rc = lib.sirius_debug_gemm(X.data_ptr(), nt, 256, W[r % ncopy].data_ptr(),
                                           W2[r % ncopy].data_ptr() if dual else None, out.data_ptr(), M, N, K)
                e1.record()
                torch.cuda.synchronize()
                assert rc == 0, rc
                if r >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            byt = N * K * 2 * (2 if dual else 1)
            med = ts[len(ts) // 2]
            print(f"{name:8s} M={M:4d} terms={nt}  median {med:7.1f} us  min {ts[0]:7.1f}  {byt / med / 1e3:7.0f} GB/s")
    del W, W2
    torch.cuda.empty_cache()
