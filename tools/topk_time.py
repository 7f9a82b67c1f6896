import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2409_03856_b200 import sirius as S
for F in (688, 3584, 14336, 28672):
    g = torch.randn((1, F), device='cuda') * 0.7
    a = torch.zeros_like(g); m = torch.zeros((1, F // 32 + 1), dtype=torch.int32, device='cuda')
    for _ in range(20): S.debug_topk(g, F // 2, a, m)
    t0 = time.perf_counter()
    for _ in range(200): S.debug_topk(g, F // 2, a, m)
    t1 = time.perf_counter()
    # empty-ish reference: a trivial torch op + sync
    for _ in range(200): g.add_(0); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(F, "topk+sync us", round((t1 - t0) / 200 * 1e6, 2), "trivial+sync us", round((t2 - t1) / 200 * 1e6, 2))
