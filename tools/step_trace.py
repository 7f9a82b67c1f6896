"""Phase timeline of the persistent decode step (globaltimer stamps per CTA, debug build path),
Llama-3-8B shape.  Not a benchmark (stamps add a __syncthreads each)."""
import os, sys
os.environ.setdefault("SIRIUS_STEP_KERNEL", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from synth import gpu as sg
from paper_2409_03856_b200 import sirius as S, driver

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
ctx = S.Sirius(cfg, sg.device_weights(cfg), synth.layer_thresholds(cfg, 0.5), batch=1, max_seq=1200, max_gamma=16)
drv = driver.Driver(ctx)
drv.begin([synth.eval_prompt(cfg, 0, 900)])
L, G = cfg.n_layers, torch.cuda.get_device_properties(0).multi_processor_count
NS = 20
buf = torch.zeros((1 + NS * L + 2, G), dtype=torch.int64, device="cuda")
ctx.graphs(False)
assert ctx.lib.sirius_debug_trace(ctx.h, buf.data_ptr()) == 1, "run with SIRIUS_STEP_KERNEL=1"
tok = torch.tensor([drv.pending[0]], dtype=torch.int32, device="cuda")
out = torch.zeros(1, dtype=torch.int32, device="cuda")
for i in range(3):
    buf.zero_()
    ctx.sparse_decode_step(tok, torch.tensor([900 + i], dtype=torch.int32, device="cuda"), 0, out)
    torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.float64)
valid = t != 0
t0 = t[0].min()
t = (t - t0) / 1e3
t[~valid] = np.nan
print(f"step: {np.nanmax(t[-1]):.1f} us")
def S_(l, k): return t[1 + l * NS + k]
# segments: (name, from slot, to slot, stat) ; from=-1 means previous layer's slot 18 (or start)
segs = [("P1 prologue", "exit_prev", 0), ("P1 rows", 0, 1), ("P1 barrier", 1, 2),
        ("P2 setup", 2, 3), ("P2 blocks", 3, 4), ("P2 group barrier", 4, 5), ("P2 combine", 5, 6), ("P2 barrier", 6, 7),
        ("P3 prologue", 7, 8), ("P3 rows", 8, 9), ("P3 barrier", 9, 10),
        ("P4 prologue", 10, 11), ("P4 gate", 11, 12), ("P4 compact", 12, 13), ("P4 up", 13, 14), ("P4 down", 14, 15),
        ("P4 barrier", 15, 16), ("P5 reduce", 16, 17), ("P5 barrier", 17, 18)]
res = {n: [] for n, _, _ in segs}
for l in range(1, L):
    for n, a, b in segs:
        ta = S_(l - 1, 18) if a == "exit_prev" else S_(l, a)
        tb = S_(l, b)
        dur = tb - ta
        res[n].append((np.nanmedian(dur), np.nanmax(dur), np.nanmax(tb) - np.nanmin(ta)))
tot = 0
for n, _, _ in segs:
    r = np.array(res[n])
    print(f"{n:18s} per-CTA median {np.median(r[:, 0]):6.2f}  max {np.median(r[:, 1]):6.2f}  span {np.median(r[:, 2]):6.2f} us")
print("layer period:", np.median(np.diff([np.nanmax(S_(l, 18)) for l in range(L)])), "us")
