"""Kernel-isolated parity of the decode CATS FFN (tier T1 of SURVEY §4) at the
Llama-3-8B and -70B layer shapes, in the launch configuration sparse_decode_step (and so bench.py)
uses: the library's FFN kernel (sirius_debug_ffn) and the oracle's layer MLP (oracle_mlp) get the
same seeded residual rows x and the same fp32 threshold t_l (PAPER.md:121 CATS threshold, readings
D2/D4), and every output is checked against an A-PRIORI fp32 error bound — no exemption:

  h2 = RMSNorm(x)             GPU fp32 (relative error <= 40 u)
  g_i = h2 . W_gate[i]        GPU: per lane n_seq = d/32 sequential fma, then a 5-level shuffle tree
  a_i = SiLU(g_i)             => |a_gpu - a_ref| <= delta_i = 1.1 (n_seq + 45) u S_i + 4 u |a_i|,
                                 S_i = sum_k |W_gate[i, k] h2_k|,  u = 2^-24
  active_i <=> |a_i| >= t_l   => identical to the oracle's mask for every neuron with
                                 ||a_ref| - t_l| > delta_i (a mismatch is only possible inside that band)
  y = sum_active m_i W_down[i], m_i = a_i (h2 . W_up[i])
                              => |y_gpu - y_ref|_k <= sum_i (|dm_i| + (n_down + G) u |m_i|) |W_down[i, k]|
                                 (+ |m_i W_down[i, k]| for a neuron inside its band that flipped),
                                 dm_i = delta_i |u_i| + |a_i| dU_i, dU_i = (n_seq + 45) u S^up_i.
The bands are computed here in fp64 from the weights (bounds, not the oracle's arithmetic); the
reference values a, mask, y come from the oracle.
"""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U = 2.0 ** -24


def _f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.fixture(scope="module", params=["8b", "70b"])
def layer_model(request):
    from synth import gpu as sg
    cfg = (synth.LLAMA3_8B if request.param == "8b" else synth.LLAMA3_70B).with_layers(1)
    wh = synth.host_weights(cfg)
    w = {k: _f64(wh[f"layers.0.{k}"]) for k in ("w_gate", "w_up", "w_down", "ffn_norm")}
    return cfg, wh, sg.device_weights(cfg), w


def _bands(cfg, w, x, a_ref, t, m_active):
    d = cfg.d_model
    h2 = x / np.sqrt(np.mean(x * x) + cfg.rms_eps) * w["ffn_norm"]
    n_seq = d // 32 + 45
    s_gate = np.abs(w["w_gate"]) @ np.abs(h2)
    delta = 1.1 * n_seq * U * s_gate + 4 * U * np.abs(a_ref)
    u = w["w_up"] @ h2
    du = n_seq * U * (np.abs(w["w_up"]) @ np.abs(h2))
    m = a_ref * u
    dm = delta * np.abs(u) + np.abs(a_ref) * du
    return delta, m, dm


@pytest.mark.parametrize("batch,atomic", [(1, True), (4, True), (8, True), (1, False), (4, False)])
def test_decode_ffn_kernel_vs_oracle(layer_model, batch, atomic, monkeypatch):
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd, w = layer_model
    if cfg.d_model == 8192 and batch == 8:
        pytest.skip("batch 8 at d = 8192 runs the row path (tensor cores), not this kernel")
    monkeypatch.setenv("SIRIUS_FFN_ATOMIC", "1" if atomic else "0")
    thr = synth.layer_thresholds(cfg, 0.5)
    t = float(thr[0])
    ctx = S.Sirius(cfg, wd, thr, batch=batch, max_seq=64, max_gamma=4)
    om = so.OracleModel(cfg, wh, max_seq=8)
    d, F = cfg.d_model, cfg.ffn_dim
    n_rows = 8 if batch == 1 else batch
    X = synth.residual_rows(100 + batch + 10 * atomic + d, n_rows, d)
    n_band = n_flip = 0
    for r0 in range(0, n_rows, batch):
        for dense in (False, True):
            x = torch.tensor(X[r0:r0 + batch], device="cuda")
            out = torch.zeros((batch, d), device="cuda")
            ga = torch.zeros((batch, F), device="cuda")
            na = torch.zeros(batch, dtype=torch.int32, device="cuda")
            ctx.debug_ffn(0, x, dense, out, ga, na)
            y_gpu, a_gpu, n_gpu = out.double().cpu().numpy(), ga.double().cpu().numpy(), na.cpu().numpy()
            for b in range(batch):
                xr = X[r0 + b].astype(np.float64)
                x_out, a_ref, mask_ref, n_ref = om.mlp(0, xr, not dense, t)
                y_ref = x_out - xr
                delta, m, dm = _bands(cfg, w, xr, a_ref, t, mask_ref)
                # a = SiLU(g) within the a-priori fp32 band
                assert np.all(np.abs(a_gpu[b] - a_ref) <= delta), float(np.max(np.abs(a_gpu[b] - a_ref) / delta))
                mask_gpu = np.ones(F, bool) if dense else np.abs(a_gpu[b]) >= t
                assert int(n_gpu[b]) == int(mask_gpu.sum())
                mis = mask_gpu != mask_ref.astype(bool)
                band = np.abs(np.abs(a_ref) - t) <= delta
                assert not np.any(mis & ~band)  # a mask difference only inside the a-priori band
                if not dense:
                    n_band += int(band.sum())
                    n_flip += int(mis.sum())
                act = mask_ref.astype(bool) | mis
                coef = np.where(act, dm + (64 + 512) * U * np.abs(m), 0.0) + np.where(mis, np.abs(m), 0.0)
                ybound = np.abs(w["w_down"]).T @ coef + 1e-30
                err = np.abs(y_gpu[b] - y_ref)
                assert np.all(err <= ybound), float(np.max(err / ybound))
                assert float(err.max()) < 1e-3 * max(1.0, float(np.abs(y_ref).max()))
    # the bands are thin: few neurons per row are even eligible to differ
    assert n_band <= 0.01 * F * n_rows, n_band
    assert n_flip <= n_band


def test_decode_ffn_kernel_bitwise_deterministic(layer_model, monkeypatch):
    """SIRIUS_FFN_ATOMIC=0 (fixed-order reduction): 10 launches, bitwise-identical outputs."""
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd, w = layer_model
    monkeypatch.setenv("SIRIUS_FFN_ATOMIC", "0")
    thr = synth.layer_thresholds(cfg, 0.5)
    ctx = S.Sirius(cfg, wd, thr, batch=1, max_seq=64, max_gamma=4)
    x = torch.tensor(synth.residual_rows(7, 1, cfg.d_model), device="cuda")
    outs = []
    for _ in range(10):
        out = torch.zeros((1, cfg.d_model), device="cuda")
        ctx.debug_ffn(0, x, False, out)
        outs.append(out.cpu())
    assert all(torch.equal(outs[0], o) for o in outs[1:])
