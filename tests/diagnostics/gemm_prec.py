"""Diagnostic: accuracy of the tcgen05 GEMM vs fp64 (relative to sum |x w|): bf16 inputs (one term)
and fp32 inputs as three bf16 terms; CUDA-core fp32 (torch, TF32 off) alongside."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2409_03856_b200 import sirius as S

torch.backends.cuda.matmul.allow_tf32 = False
g = torch.Generator(device="cpu").manual_seed(0)
for (M, N, K) in ((16, 1024, 4096), (16, 1024, 14336), (128, 1024, 4096)):
    X32 = torch.randn(M, K, generator=g)
    W = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16)
    t0 = X32.to(torch.bfloat16); r1 = X32 - t0.float(); t1 = r1.to(torch.bfloat16); t2 = (r1 - t1.float()).to(torch.bfloat16)
    X3 = torch.stack([t0, t1, t2])
    scale = (X32.double().abs() @ W.double().abs().T)
    for name, Xin, xref in (("bf16 x, 1 term", t0.cuda(), t0.double()), ("fp32 x, 3 terms", X3.cuda(), X32.double()),
                            ("fp32 x, 2 terms", X3[:2].contiguous().cuda(), X32.double())):
        out = torch.zeros((M, N), device="cuda")
        S.debug_gemm(Xin, W.cuda(), out, M)
        ref = xref @ W.double().T
        e = ((out.double().cpu() - ref).abs() / scale)
        print(f"M{M} N{N} K{K} {name}: max err/sum|xw| {e.max():.2e}, median {e.median():.2e}", flush=True)
    c = (X32.cuda() @ W.float().cuda().T).double().cpu()
    e = ((c - X32.double() @ W.double().T).abs() / scale)
    print(f"   torch fp32 CUDA cores: max {e.max():.2e}, median {e.median():.2e}", flush=True)
