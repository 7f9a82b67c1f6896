"""The decode GEMV kernel (gemv_ffn.cu) in isolation against an fp64
product of the same bf16 weights and fp32 activations, over the shapes the decode path uses (ragged
per-CTA row ranges, K from the tiny model's 256 to Llama-3-70B's 8192), its three prologues and the
packed lowest-index argmax epilogue."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,K,B", [(512, 256, 1), (6144, 4096, 1), (4096, 4096, 2), (1000, 4096, 4),
                                      (2304, 8192, 1), (151, 512, 1), (16032, 4096, 1)])
def test_gemv_vs_fp64(rows, K, B):
    from paper_2409_03856_b200 import sirius as S
    g = torch.Generator(device="cuda").manual_seed(rows + K + B)
    W = (torch.randn(rows, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    x = torch.randn(B, K, device="cuda", generator=g)
    out = torch.full((B, rows), float("nan"), device="cuda")
    am = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    S.debug_gemv(W, x, out, am)
    ref = x.double() @ W.double().T
    err = (out.double() - ref).abs()
    bound = 64 * 2.0 ** -24 * (x.double().abs() @ W.double().abs().T)  # fp32 accumulation, K-term sums
    assert bool(torch.all(err <= bound + 1e-30)), float((err / (bound + 1e-30)).max())
    # argmax over the kernel's own fp32 outputs, lowest index on ties
    o = out.cpu().numpy()
    for b in range(B):
        assert int(am[b]) == int(np.flatnonzero(o[b] == o[b].max())[0])


def test_gemv_argmax_tie_lowest_index():
    from paper_2409_03856_b200 import sirius as S
    K, rows = 4096, 6000
    W = torch.zeros(rows, K, device="cuda", dtype=torch.bfloat16)
    W[[777, 4000, 5999], :] = 1.0
    x = torch.ones(1, K, device="cuda")
    out = torch.zeros(1, rows, device="cuda")
    am = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    S.debug_gemv(W, x, out, am)
    assert int(am[0]) == 777


def _rms(x, w, eps=1e-5):
    return x / torch.sqrt((x * x).mean(dim=1, keepdim=True) + eps) * w


@pytest.mark.parametrize("mode", ["resid", "embed"])
@pytest.mark.parametrize("rows,K,B", [(512, 256, 1), (6144, 4096, 1), (4096, 4096, 2)])
def test_gemv_prologues(mode, rows, K, B):
    """Residual add + RMSNorm and embedding-gather + RMSNorm prologues (D15: fp32 h)."""
    from paper_2409_03856_b200 import sirius as S
    g = torch.Generator(device="cuda").manual_seed(7 * rows + K + B)
    W = (torch.randn(rows, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    nw = (1 + 0.1 * torch.randn(K, device="cuda", generator=g)).to(torch.bfloat16)
    out = torch.full((B, rows), float("nan"), device="cuda")
    if mode == "resid":
        x = torch.randn(B, K, device="cuda", generator=g)
        dl = torch.randn(B, K, device="cuda", generator=g)
        res = torch.zeros(B, K, device="cuda")
        S.debug_gemv(W, x, out, delta=dl, norm_w=nw, res_out=res)
        xs = x.double() + dl.double()
        assert torch.equal(res, x + dl)
    else:
        E = torch.randn(300, K, device="cuda", generator=g).to(torch.bfloat16)
        tok = torch.tensor([5, 299, 0, 17][:B], dtype=torch.int32, device="cuda")
        res = torch.zeros(B, K, device="cuda")
        S.debug_gemv(W, None, out, norm_w=nw, tokens=tok, embed=E, res_out=res)
        xs = E.double()[tok.long()]
        assert torch.equal(res, E.float()[tok.long()])  # the embedding row is the layer-0 residual
    h = _rms(xs, nw.double())
    ref = h @ W.double().T
    bound = 64 * 2.0 ** -24 * (h.abs() @ W.double().abs().T) + 1e-6 * ref.abs().max()
    err = (out.double() - ref).abs()
    assert bool(torch.all(err <= bound)), float((err / bound).max())
