"""GPU parity of top-k FSparse (PAPER.md:121 footnote; reading D30) against the oracle
through the C ABI (sirius_topk_enable + sparse_decode_step(SIRIUS_TOPK)):
  * the selection is exact: the oracle's top-k rule applied to the GPU's own exported a (fp32) gives the
    GPU's active set bit for bit (exactly k per layer);
  * against the oracle's fp64 a, sets differ only at neurons within the float error of the k-th |a|;
  * logits agree within the north-star tolerance while the sets agree;
  * the Sirius loop over the top-k draft model is token-exact (tiny, free running)."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ABS, REL = 2e-2, 1e-2


def _ctx(cfg, thr, keep, batch=1, max_seq=512, gamma=16):
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    ctx = S.Sirius(cfg, sg.device_weights(cfg), thr, batch=batch, max_seq=max_seq, max_gamma=gamma)
    ctx.sirius_topk_enable(keep)
    return ctx


def _topk_mask(a, keep):
    F = a.size
    k = so.csparse_keep_count(F, keep)
    order = sorted(range(F), key=lambda i: (-abs(float(a[i])), i))
    m = np.zeros(F, dtype=bool)
    m[order[:k]] = True
    return m


@pytest.mark.parametrize("model,P", [("tiny", 64), ("8b1l", 200)])
def test_topk_decode_lockstep(model, P):
    from paper_2409_03856_b200 import sirius as S
    cfg = synth.TINY if model == "tiny" else synth.LLAMA3_8B.with_layers(1)
    wh = synth.host_weights(cfg)
    thr = synth.layer_thresholds(cfg, 0.5)
    keep = 0.5
    ctx = _ctx(cfg, thr, keep)
    om = so.OracleModel(cfg, wh, max_seq=512, max_gamma=16)
    prompt = synth.eval_prompt(cfg, 4, P)
    first = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(torch.tensor(prompt, device="cuda"), [P], first)
    tok = so.argmax_lowest(om.prefill_last(prompt))
    L, F = cfg.n_layers, cfg.ffn_dim
    k = so.csparse_keep_count(F, keep)
    topk = np.full(L, keep, dtype=np.float32)
    for step in range(3):
        pos = P + step
        r = om.decode(tok, pos, True, topk=topk, want_gate=True, want_mask=True)
        ti = torch.tensor([tok], dtype=torch.int32, device="cuda")
        pi = torch.tensor([pos], dtype=torch.int32, device="cuda")
        to = torch.zeros(1, dtype=torch.int32, device="cuda")
        lo = torch.zeros((1, cfg.vocab), device="cuda")
        na = torch.zeros((1, L), dtype=torch.int32, device="cuda")
        ga = torch.zeros((1, L, F), device="cuda")
        ctx.sparse_decode_step(ti, pi, S.SIRIUS_TOPK, to, lo, na, ga)
        a_gpu = ga.cpu().numpy()[0]
        assert np.all(na.cpu().numpy()[0] == k)
        same_sets = True
        for l in range(L):
            m_gpu = _topk_mask(a_gpu[l], keep)  # the oracle's rule on the GPU's a: must be the GPU's set
            kth = np.sort(np.abs(r.gate[l]))[::-1][k - 1]
            diff = m_gpu != r.mask[l].astype(bool)
            err = np.abs(a_gpu[l] - r.gate[l])
            band = np.abs(np.abs(r.gate[l]) - kth) <= 2 * err.max() + 1e-7
            assert not np.any(diff & ~band), np.flatnonzero(diff & ~band)[:8]
            same_sets &= not diff.any()
        if same_sets:
            e = np.abs(lo.cpu().numpy()[0] - r.logits)
            assert np.all(e <= ABS + REL * np.abs(r.logits)), float(e.max())
        tok = so.argmax_lowest(r.logits)


def test_topk_gpu_set_is_the_rule_on_its_own_activations():
    """Kernel-level: decode with gate export; the set the FFN used (n_active) and the exported a agree
    with the exact top-k rule on those a (bit-exact selection, ties to the lower index)."""
    from paper_2409_03856_b200 import sirius as S
    cfg = synth.TINY
    thr = synth.layer_thresholds(cfg, 0.5)
    for keep in (0.25, 0.5, 0.75):
        ctx = _ctx(cfg, thr, keep)
        prompt = synth.eval_prompt(cfg, 1, 32)
        first = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.sirius_prefill(torch.tensor(prompt, device="cuda"), [32], first)
        lo = torch.zeros((1, cfg.vocab), device="cuda")
        na = torch.zeros((1, cfg.n_layers), dtype=torch.int32, device="cuda")
        ga = torch.zeros((1, cfg.n_layers, cfg.ffn_dim), device="cuda")
        to = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.sparse_decode_step(first, torch.tensor([32], dtype=torch.int32, device="cuda"), S.SIRIUS_TOPK, to, lo, na,
                               ga)
        assert np.all(na.cpu().numpy()[0] == so.csparse_keep_count(cfg.ffn_dim, keep))


@pytest.mark.parametrize("r", [0.1, 0.3])
def test_topk_sirius_free_running_token_exact(r):
    from paper_2409_03856_b200 import driver
    cfg = synth.TINY
    wh = synth.host_weights(cfg)
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 2, 64)
    ref = so.generate(so.OracleModel(cfg, wh, max_seq=512, max_gamma=16), prompt, 32, 4, r, thr, topk_keep=0.5)
    out = driver.Driver(_ctx(cfg, thr, 0.5), topk=True).sirius([prompt], 32, 4, r)
    assert out.tokens[0] == ref.tokens
    assert out.advances(0) == ref.advances[:len(out.kernels)]


@pytest.mark.parametrize("F,k,ties", [(14336, 7168, 0), (14336, 7168, 40), (28672, 1000, 7), (688, 344, 5),
                                      (100, 1, 0), (3000, 3000, 0)])
def test_topk_select_kernel_exact_with_forced_ties(F, k, ties):
    """The selection kernel alone (both of its paths): with `ties` > 0 several neurons get exactly the
    k-th largest |a| (the lowest-index ones must win), else the k-th value is unique.  The mask must
    be the rule applied to the kernel's own a (bit-exact)."""
    from paper_2409_03856_b200 import sirius as S
    rng = np.random.default_rng(F + k + ties)
    g = rng.standard_normal((2, F)).astype(np.float32) * 0.7
    for b in range(2):
        if ties:
            a = g[b] / (1.0 + np.exp(-g[b].astype(np.float64)))
            kth = np.sort(np.abs(a))[::-1][k - 1]
            j = int(np.argmin(np.abs(np.abs(a) - kth)))
            idx = rng.choice(F, size=ties, replace=False)
            g[b, idx] = g[b, j]  # same g -> same a (same kernel arithmetic) -> a tie at the boundary
    gd = torch.tensor(g, device="cuda")
    ad = torch.zeros_like(gd)
    md = torch.zeros((2, F // 32 + 1), dtype=torch.int32, device="cuda")
    S.debug_topk(gd, k, ad, md)
    a = ad.cpu().numpy()
    m = md.cpu().numpy().view(np.uint32)
    for b in range(2):
        order = np.lexsort((np.arange(F), -np.abs(a[b]).astype(np.float64)))
        want = np.zeros(F, dtype=bool)
        want[order[:k]] = True
        got = ((m[b][np.arange(F) >> 5] >> (np.arange(F) & 31)) & 1).astype(bool)
        assert got.sum() == k
        np.testing.assert_array_equal(got, want)
