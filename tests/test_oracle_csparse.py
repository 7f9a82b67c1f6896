"""Pins for the oracle's CSparse (Griffin-style coarse-grained sparsity) part — SURVEY.md §8(f) N2,
PAPER.md:62 (§2.1: "within the same input prompt, the sparsity pattern is fixed for all tokens
generated"), :182 (§3.2: the pattern is predetermined after prefilling, so the gate is sparsified
too), :471 (Griffin, the paper's latency setting).  Reading D28: statistic = sum over the
prompt of |SiLU(g)| per neuron, keep round(keep * ffn) (halves up) per layer, ties to the lower index.
CPU only."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

from test_oracle_pins import _f64, _hf_full_fp64, _hf_llama


def test_csparse_stats_match_hf_llama_activations(tiny, monkeypatch):
    """The statistic equals sum_p |act_fn(gate_proj(post_attention_layernorm(x_p)))| taken from
    transformers.LlamaForCausalLM (fp64, hooks on the MLP activation) over the same prompt."""
    torch = pytest.importorskip("torch")
    cfg, w = tiny
    m = _hf_llama(cfg, w)
    _hf_full_fp64(monkeypatch, m, cfg)
    prompt = synth.eval_prompt(cfg, 4, 40)
    acts = {}

    def hook(l):
        def f(mod, inp, out):
            acts[l] = out[0].abs().sum(0).numpy()  # [ffn]: sum over prompt positions
        return f

    hs = [m.model.layers[l].mlp.act_fn.register_forward_hook(hook(l)) for l in range(cfg.n_layers)]
    with torch.no_grad():
        m(torch.tensor(prompt[None].astype(np.int64)))
    for h in hs:
        h.remove()
    _, stats = so.OracleModel(cfg, w, max_seq=64, round_kv=False).prefill_stats(prompt)
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(stats[l], acts[l], rtol=1e-9, atol=1e-9)


def test_csparse_plan_selection_brute_force():
    """Top-k by the statistic, ties to the lower index, |set| = round(keep * ffn) (halves up), and the
    set at a smaller keep is a subset of the set at a larger keep."""
    rng = np.random.default_rng(11)
    F = 37
    s = rng.integers(0, 9, size=(3, F)).astype(np.float64)  # many exact ties
    for keep in (0.1, 0.25, 0.5, 0.7, 1.0):
        k = so.csparse_keep_count(F, keep)
        assert k == int(keep * F + 0.5)
        plan = so.csparse_plan(s, keep)
        for l in range(3):
            brute = sorted(range(F), key=lambda i: (-s[l, i], i))[:k]  # pure-Python definition
            assert sorted(np.flatnonzero(plan[l]).tolist()) == sorted(brute)
    for lo, hi in ((0.25, 0.5), (0.5, 0.7)):
        assert np.all(so.csparse_plan(s, lo) <= so.csparse_plan(s, hi))
    assert so.csparse_keep_count(688, 0.5) == 344 and so.csparse_keep_count(5, 0.5) == 3


def test_csparse_mlp_equals_dense_mlp_with_unplanned_neurons_zeroed(tiny):
    """Brute force: the CSparse MLP equals the dense MLP on weights whose W_gate, W_up and
    W_down rows outside the plan are zeroed — exact (the gate is sparsified too)."""
    cfg, w = tiny
    rng = np.random.default_rng(12)
    m = so.OracleModel(cfg, w, max_seq=8)
    plan = np.zeros(cfg.ffn_dim, dtype=np.uint8)
    plan[rng.permutation(cfg.ffn_dim)[:300]] = 1
    x = rng.standard_normal(cfg.d_model) * 2.0
    for l in range(cfg.n_layers):
        xs, _, mask, n = m.mlp(l, x, True, plan=plan)
        assert n == 300 and np.array_equal(mask, plan)
        w2 = dict(w)
        for name in ("w_gate", "w_up", "w_down"):
            z = w[f"layers.{l}.{name}"].copy()
            z[plan == 0] = 0
            w2[f"layers.{l}.{name}"] = z
        xd, _, _, _ = so.OracleModel(cfg, w2, max_seq=8).mlp(l, x, False)
        np.testing.assert_array_equal(xs, xd)
        # and the numpy form of the restricted MLP
        mr = so.OracleModel(cfg, w, max_seq=8, round_kv=False)
        h = x / np.sqrt(np.mean(x * x) + cfg.rms_eps) * _f64(w[f"layers.{l}.ffn_norm"])
        sel = plan.astype(bool)
        g = _f64(w[f"layers.{l}.w_gate"])[sel] @ h
        u = _f64(w[f"layers.{l}.w_up"])[sel] @ h
        ref = x + _f64(w[f"layers.{l}.w_down"])[sel].T @ (g / (1 + np.exp(-g)) * u)
        np.testing.assert_allclose(mr.mlp(l, x, True, plan=plan)[0], ref, rtol=1e-11, atol=1e-11)


def test_csparse_keep_one_equals_dense(tiny):
    """keep = 1: the plan keeps every neuron and the CSparse model is the dense model — bitwise."""
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 5, 20)
    om = so.OracleModel(cfg, w, max_seq=64)
    _, stats = om.prefill_stats(prompt)
    plan = so.csparse_plan(stats, 1.0)
    assert plan.all()
    r1 = om.decode(9, 20, True, plan=plan)
    om2 = so.OracleModel(cfg, w, max_seq=64)
    om2.prefill(prompt)
    r2 = om2.decode(9, 20, False)
    np.testing.assert_array_equal(r1.logits, r2.logits)


def test_csparse_sirius_generate_accounting(tiny):
    """CSparse Sirius loop: the plan is the prompt's, fixed for the generation; r = 0 accepts every
    draft; EXACT_ARGMAX reproduces dense greedy (the correction is lossless in that mode)."""
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 6, 24)
    res = so.generate(so.OracleModel(cfg, w, max_seq=128), prompt, 20, 4, 0.0, None, csparse_keep=0.5)
    assert res.plan is not None and int(res.plan[0].sum()) == so.csparse_keep_count(cfg.ffn_dim, 0.5)
    assert all(a == 4 for a in res.advances[:-1])
    ex = so.generate(so.OracleModel(cfg, w, max_seq=128), prompt, 20, 4, 0.0, None,
                     accept_mode=so.ACCEPT_EXACT_ARGMAX, csparse_keep=0.5)
    dense = so.greedy_decode(so.OracleModel(cfg, w, max_seq=128), prompt, 20)
    assert ex.tokens == dense


# ------------------------------------------------------------------ top-k FSparse
def test_topk_fsparse_mlp_brute_force(tiny):
    """Top-k FSparse (PAPER.md:121 footnote "topk on the Gate Layer activations", reading D30): exactly
    round(keep * ffn) neurons, the largest |SiLU(g)| with exact ties to the lower index (pure-Python
    sort of the oracle's own exported a), and the MLP equals the dense MLP with the other up/down rows
    zeroed."""
    cfg, w = tiny
    m = so.OracleModel(cfg, w, max_seq=8)
    rng = np.random.default_rng(21)
    x = rng.standard_normal(cfg.d_model) * 2.0
    for keep in (0.3, 0.5):
        for l in range(cfg.n_layers):
            xs, a, mask, n = m.mlp(l, x, True, topk=keep)
            k = so.csparse_keep_count(cfg.ffn_dim, keep)
            assert n == k == int(mask.sum())
            brute = sorted(range(cfg.ffn_dim), key=lambda i: (-abs(a[i]), i))[:k]
            assert sorted(np.flatnonzero(mask).tolist()) == sorted(brute)
            w2 = dict(w)
            for name in ("w_up", "w_down"):
                z = w[f"layers.{l}.{name}"].copy()
                z[mask == 0] = 0
                w2[f"layers.{l}.{name}"] = z
            xd, _, _, _ = so.OracleModel(cfg, w2, max_seq=8).mlp(l, x, False)
            np.testing.assert_array_equal(xs, xd)


def test_topk_keep_one_equals_dense(tiny):
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 8, 16)
    m1, m2 = so.OracleModel(cfg, w, max_seq=32), so.OracleModel(cfg, w, max_seq=32)
    m1.prefill(prompt)
    m2.prefill(prompt)
    r1 = m1.decode(3, 16, True, topk=np.ones(cfg.n_layers, dtype=np.float32), want_mask=True)
    r2 = m2.decode(3, 16, False)
    assert r1.mask.all()
    np.testing.assert_array_equal(r1.logits, r2.logits)


# ------------------------------------------------------------------ sampled decoding (reading D31)
def test_splitmix64_reference_values():
    """The counter-based generator is SplitMix64's output function: the published sequence of the
    generator seeded with 0 starts e220a8397b1dcdaf, 6e789e6aa1b965f4."""
    assert so.splitmix64(0) == 0xE220A8397B1DCDAF
    assert so.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    u = [so.sample_uniform(7, 0, p) for p in range(2000)]
    assert all(0.0 <= x < 1.0 for x in u) and abs(np.mean(u) - 0.5) < 0.02
    assert all(x * 16777216.0 == int(x * 16777216.0) for x in u[:50])  # 24-bit values (exact in fp32)


def test_sampler_inverse_cdf_brute_force():
    """Over an evenly spaced grid of u, each token is drawn with frequency softmax(l / T)_v (to the grid
    resolution); T -> 0 gives the argmax."""
    rng = np.random.default_rng(31)
    l = rng.standard_normal(37) * 3.0
    for T in (0.6, 1.0):
        n = 1 << 15
        counts = np.bincount([so.sample_token(l, T, (i + 0.5) / n) for i in range(n)], minlength=l.size)
        p = np.exp((l - l.max()) / T)
        p /= p.sum()
        assert np.max(np.abs(counts / n - p)) <= 2.0 / n
    assert so.sample_token(l, 1e-3, 0.999) == so.argmax_lowest(l)


def test_sampled_sirius_accounting(tiny):
    """Sampled Sirius (temperature 0.6): r = 0 accepts every draft; the run is a function of the seed."""
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 9, 24)
    a = so.generate(so.OracleModel(cfg, w, max_seq=128), prompt, 20, 4, 0.0, thr, temperature=0.6, seed=3)
    b = so.generate(so.OracleModel(cfg, w, max_seq=128), prompt, 20, 4, 0.0, thr, temperature=0.6, seed=3)
    c = so.generate(so.OracleModel(cfg, w, max_seq=128), prompt, 20, 4, 0.0, thr, temperature=0.6, seed=4)
    assert a.tokens == b.tokens and a.tokens != c.tokens
    assert all(x == 4 for x in a.advances[:-1])
