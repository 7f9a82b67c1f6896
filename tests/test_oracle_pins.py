"""Pins for the CPU oracle (oracle/): each test checks the oracle against something other than
itself — a library model, a brute-force formula, an invariant the paper fixes, or a number the
paper prints.  CPU only (no GPU marker)."""
import csv
import json
import os

import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ------------------------------------------------------------------ dense decoder vs HuggingFace
def _hf_llama(cfg, w):
    """transformers.LlamaForCausalLM in fp64 carrying the synthetic weights."""
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    hc = tr.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.ffn_dim,
                        num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                        num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rope_theta=cfg.rope_theta,
                        rms_norm_eps=cfg.rms_eps, max_position_embeddings=4096, tie_word_embeddings=False,
                        attention_bias=False, mlp_bias=False)
    torch.manual_seed(0)
    m = tr.LlamaForCausalLM(hc).to(torch.float64).eval()
    t = lambda a: torch.from_numpy(_f64(a))
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    sd = {"model.embed_tokens.weight": t(w["embed"]), "model.norm.weight": t(w["final_norm"]),
          "lm_head.weight": t(w["lm_head"])}
    for l in range(cfg.n_layers):
        p = f"model.layers.{l}."
        q = t(w[f"layers.{l}.w_qkv"])
        sd[p + "self_attn.q_proj.weight"] = q[:H * hd]
        sd[p + "self_attn.k_proj.weight"] = q[H * hd:(H + KV) * hd]
        sd[p + "self_attn.v_proj.weight"] = q[(H + KV) * hd:]
        sd[p + "self_attn.o_proj.weight"] = t(w[f"layers.{l}.w_o"])
        sd[p + "mlp.gate_proj.weight"] = t(w[f"layers.{l}.w_gate"])
        sd[p + "mlp.up_proj.weight"] = t(w[f"layers.{l}.w_up"])
        sd[p + "mlp.down_proj.weight"] = t(w[f"layers.{l}.w_down"]).T.contiguous()
        sd[p + "input_layernorm.weight"] = t(w[f"layers.{l}.attn_norm"])
        sd[p + "post_attention_layernorm.weight"] = t(w[f"layers.{l}.ffn_norm"])
    res = m.load_state_dict(sd, strict=False)
    assert not res.missing_keys and not res.unexpected_keys
    return m


def test_dense_decoder_matches_hf_llama_fp64(tiny, monkeypatch):
    """The dense decoder (embed, RMSNorm, RoPE rotate-half, GQA kv=h//(H/KV), SiLU-gated MLP, head)
    equals transformers.LlamaForCausalLM in fp64 with the same weights (oracle with no activation
    rounding of the KV cache): to fp64 summation-order error once HF's fp32 RMSNorm / softmax / RoPE
    table are made fp64 (and D16's table); with HF's stock fp32 pieces, to ~1e-5."""
    torch = pytest.importorskip("torch")
    cfg, w = tiny
    m = _hf_llama(cfg, w)
    prompt = synth.eval_prompt(cfg, 0, 48)
    with torch.no_grad():
        stock = m(torch.tensor(prompt[None].astype(np.int64))).logits[0].numpy()
    _hf_full_fp64(monkeypatch, m, cfg)
    prompt = synth.eval_prompt(cfg, 0, 48)
    with torch.no_grad():
        ref = m(torch.tensor(prompt[None].astype(np.int64))).logits[0].numpy()
    om = so.OracleModel(cfg, w, max_seq=64, round_kv=False)
    mine = om.prefill(prompt)
    assert np.abs(ref).max() > 5.0  # logits are not degenerate
    assert np.abs(mine - ref).max() < 1e-9, np.abs(mine - ref).max()
    assert np.abs(mine - stock).max() < 5e-5, np.abs(mine - stock).max()


def _hf_full_fp64(monkeypatch, m, cfg):
    """HF computes RMSNorm, the attention softmax and the RoPE table in fp32 even for an fp64 model;
    make the first two fp64 and the table that of reading D16 (angles in fp64, cos/sin rounded to
    fp32) — precision conventions of the library, not part of the method — and select eager
    attention."""
    import torch
    from transformers.models.llama import modeling_llama as ml
    hd, half = cfg.head_dim, cfg.head_dim // 2

    def rope_d16(x, position_ids):
        inv = cfg.rope_theta ** (-2.0 * torch.arange(half, dtype=torch.float64) / hd)
        ang = position_ids[0].to(torch.float64)[:, None] * inv[None, :]
        c = torch.cos(ang).to(torch.float32).to(torch.float64)
        s = torch.sin(ang).to(torch.float32).to(torch.float64)
        return torch.cat([c, c], -1)[None], torch.cat([s, s], -1)[None]
    monkeypatch.setattr(m.model.rotary_emb, "forward", rope_d16)

    def rms_fp64(self, x):
        return self.weight * (x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.variance_epsilon))

    def eager_fp64(module, query, key, value, attention_mask, scaling, dropout=0.0, **kw):
        k = ml.repeat_kv(key, module.num_key_value_groups)
        v = ml.repeat_kv(value, module.num_key_value_groups)
        s = torch.matmul(query, k.transpose(2, 3)) * scaling
        if attention_mask is not None:
            s = s + attention_mask
        p = torch.softmax(s, dim=-1)
        return torch.matmul(p, v).transpose(1, 2).contiguous(), p
    monkeypatch.setattr(ml.LlamaRMSNorm, "forward", rms_fp64)
    monkeypatch.setattr(ml, "eager_attention_forward", eager_fp64)
    m.config._attn_implementation = "eager"
    for layer in m.model.layers:
        layer.self_attn.config._attn_implementation = "eager"


def _rne_bf16(t):
    """fp64 tensor -> nearest bf16 value (ties to even), computed in fp64 (no fp32 double rounding)."""
    import torch
    m, e = torch.frexp(t)
    return torch.ldexp(torch.round(torch.ldexp(m, torch.full_like(e, 8))), e - 8)


@pytest.mark.parametrize("variant", ["oracle_reading", "k_rounded_before_rope", "q_rounded_too", "no_rounding"])
def test_kv_bf16_rounding_placement_against_hf(tiny, monkeypatch, variant):
    """Pins WHERE the oracle rounds to bf16 (D15: the stored K after RoPE and V, nothing
    else) against HuggingFace LlamaForCausalLM in fp64, with a KV cache whose update() stores bf16
    values of the post-RoPE K and V, and the RoPE table of reading D16 (angles in fp64, cos/sin
    rounded to fp32).  The oracle (round_kv) must equal that model to fp64 summation-order error;
    the three mis-placed variants (K rounded before RoPE; q rounded as well; nothing rounded) must
    all differ from the oracle by far more — so a misplaced rounding in the oracle fails this test."""
    torch = pytest.importorskip("torch")
    from transformers import DynamicCache
    from transformers.models.llama import modeling_llama as ml
    cfg, w = tiny
    m = _hf_llama(cfg, w)
    _hf_full_fp64(monkeypatch, m, cfg)
    orig_rope = ml.apply_rotary_pos_emb

    class RoundingCache(DynamicCache):
        def update(self, k, v, layer_idx, *a, **kw):
            if variant in ("oracle_reading", "q_rounded_too"):
                k, v = _rne_bf16(k), _rne_bf16(v)
            return super().update(k, v, layer_idx, *a, **kw)

    def rope_variant(q, k, cos, sin, *a, **kw):
        if variant == "k_rounded_before_rope":
            k = _rne_bf16(k)
        q2, k2 = orig_rope(q, k, cos, sin, *a, **kw)
        if variant == "q_rounded_too":
            q2 = _rne_bf16(q2)
        return q2, k2
    monkeypatch.setattr(ml, "apply_rotary_pos_emb", rope_variant)
    if variant == "k_rounded_before_rope":  # V is not rotated: round it where it is produced
        for layer in m.model.layers:
            layer.self_attn.v_proj.register_forward_hook(lambda mod, inp, out: _rne_bf16(out))
    prompt = synth.eval_prompt(cfg, 0, 48)
    with torch.no_grad():
        ref = m(torch.tensor(prompt[None].astype(np.int64)), past_key_values=RoundingCache(),
                use_cache=True).logits[0].numpy()
    mine = so.OracleModel(cfg, w, max_seq=64, round_kv=True).prefill(prompt)
    diff = float(np.abs(mine - ref).max())
    print(f"{variant}: max |oracle - HF| = {diff:.3e}")
    if variant == "oracle_reading":
        assert diff < 1e-9, diff
    else:
        assert diff > 1e-4, (variant, diff)


def test_round_bf16_is_rne():
    """round_bf16 = round-to-nearest-even at 8 significant bits (torch's fp32->bf16 cast is RNE)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(5000) * 10.0 ** rng.integers(-6, 6, 5000),
                        # exact ties: 1 + k/256 + 1/512 (halfway between bf16 neighbours)
                        1.0 + np.arange(16) / 128.0 + 1.0 / 256.0]).astype(np.float32).astype(np.float64)
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    mine = np.array([so.round_bf16(v) for v in x])
    np.testing.assert_array_equal(mine, ref)
    assert so.round_bf16(1.0 + 1.0 / 256.0) == 1.0  # tie -> even
    assert so.round_bf16(1.0 + 3.0 / 256.0) == 1.0 + 4.0 / 256.0


# ------------------------------------------------------------------ cache / chunk invariants
def test_kv_identity_and_chunk_equals_sequential(tiny):
    """SPEC S:60/S:83 (KV-cache identity) and S:79/S:84 (chunk == sequential): incremental decode
    rows equal the prefill rows, and the verify pass over a kernel (staging) equals sequential dense
    decode of the same tokens — bitwise, since every row's arithmetic is row-independent."""
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 1, 40)
    a = so.OracleModel(cfg, w, max_seq=64, max_gamma=8)
    full = a.prefill(prompt)
    b = so.OracleModel(cfg, w, max_seq=64, max_gamma=8)
    b.prefill(prompt[:30])
    inc = np.stack([b.decode(int(t), 30 + i, False).logits for i, t in enumerate(prompt[30:])])
    np.testing.assert_array_equal(inc, full[30:])
    c = so.OracleModel(cfg, w, max_seq=64, max_gamma=8)
    c.prefill(prompt[:32])
    lf = c.verify([int(t) for t in prompt[32:40]], 32)
    np.testing.assert_array_equal(lf, full[32:40])
    # the verify pass did not touch the cache: rows >= 32 are still unwritten (zero)
    k, _ = c.read_cache(0, 40)
    assert np.all(k[32:] == 0) and np.any(k[:32] != 0)


def test_prefill_last_writes_the_same_cache_as_prefill(tiny):
    """prefill_last (K/V-only rows for all but the last prompt position) leaves the cache and the
    last logits bitwise equal to the full prefill: the skipped work does not feed them."""
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 4, 37)
    a = so.OracleModel(cfg, w, max_seq=64, max_gamma=8)
    full = a.prefill(prompt)
    b = so.OracleModel(cfg, w, max_seq=64, max_gamma=8)
    last = b.prefill_last(prompt)
    np.testing.assert_array_equal(last, full[-1])
    for l in range(cfg.n_layers):
        for x, y in zip(a.read_cache(l, 37), b.read_cache(l, 37)):
            np.testing.assert_array_equal(x, y)


def test_rewrite_equivalence(tiny):
    """SPEC S:147 / S:553: after kv_rewrite the cache rows [0,len) equal those of a
    dense prefill of the committed tokens, bitwise."""
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.1)
    prompt = synth.eval_prompt(cfg, 2, 32)
    m = so.OracleModel(cfg, w, max_seq=128, max_gamma=8)
    res = so.generate(m, prompt, 20, 5, 0.6, thr)
    committed = list(prompt) + res.all_tokens[:-1]  # the last token is pending (no K/V yet)
    n = len(prompt) + sum(res.advances)
    ref = so.OracleModel(cfg, w, max_seq=128, max_gamma=8)
    ref.prefill(committed[:n])
    for l in range(cfg.n_layers):
        k1, v1 = m.read_cache(l, n)
        k2, v2 = ref.read_cache(l, n)
        np.testing.assert_array_equal(k1, k2)
        np.testing.assert_array_equal(v1, v2)


# ------------------------------------------------------------------ CATS MLP
def test_sparse_mlp_equals_dense_mlp_with_inactive_neurons_zeroed(tiny):
    """Brute force: the CATS MLP equals the dense MLP on weights whose inactive W_up rows
    and W_down rows are zeroed — exact."""
    cfg, w = tiny
    thr = float(synth.cats_threshold(0.5))
    rng = np.random.default_rng(3)
    m = so.OracleModel(cfg, w, max_seq=8)
    for trial in range(3):
        x = rng.standard_normal(cfg.d_model) * 2.0
        for l in range(cfg.n_layers):
            xs, a, mask, n = m.mlp(l, x, True, thr)
            assert 0.3 * cfg.ffn_dim < n < 0.7 * cfg.ffn_dim
            assert n == mask.sum() and np.array_equal(mask.astype(bool), np.abs(a) >= thr)
            w2 = dict(w)
            up = w[f"layers.{l}.w_up"].copy()
            dn = w[f"layers.{l}.w_down"].copy()
            up[mask == 0] = 0
            dn[mask == 0] = 0
            w2[f"layers.{l}.w_up"], w2[f"layers.{l}.w_down"] = up, dn
            m2 = so.OracleModel(cfg, w2, max_seq=8)
            xd, _, mask_d, nd = m2.mlp(l, x, False)
            assert nd == cfg.ffn_dim and mask_d.all()
            np.testing.assert_array_equal(xs, xd)


def test_mlp_formula_against_numpy(tiny):
    """The MLP equals x + W_down^T (SiLU(W_gate h) * W_up h * mask) written
    with numpy matrix products, h = x / sqrt(mean x^2 + eps) * w_norm.  Catches a transposed operand,
    a wrong activation or a wrong norm."""
    cfg, w = tiny
    m = so.OracleModel(cfg, w, max_seq=8, round_kv=False)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(cfg.d_model)
    thr = float(synth.cats_threshold(0.4))
    for l in range(cfg.n_layers):
        h = x / np.sqrt(np.mean(x * x) + cfg.rms_eps) * _f64(w[f"layers.{l}.ffn_norm"])
        g = _f64(w[f"layers.{l}.w_gate"]) @ h
        a = g / (1.0 + np.exp(-g))
        mask = np.abs(a) >= thr
        u = _f64(w[f"layers.{l}.w_up"]) @ h
        ref = x + _f64(w[f"layers.{l}.w_down"]).T @ (a * u * mask)
        xs, a_o, mask_o, _ = m.mlp(l, x, True, thr)
        np.testing.assert_allclose(a_o, a, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(mask_o.astype(bool), mask)
        np.testing.assert_allclose(xs, ref, rtol=1e-11, atol=1e-11)


def test_threshold_zero_sparse_equals_dense(tiny):
    """north_star: threshold 0 (density 1) makes the sparse model equal the dense model — bitwise."""
    cfg, w = tiny
    prompt = synth.eval_prompt(cfg, 3, 24)
    zero = np.zeros(cfg.n_layers, dtype=np.float32)
    a = so.greedy_decode(so.OracleModel(cfg, w, max_seq=64), prompt, 12, sparse=True, thresholds=zero)
    b = so.greedy_decode(so.OracleModel(cfg, w, max_seq=64), prompt, 12, sparse=False)
    assert a == b
    m1, m2 = so.OracleModel(cfg, w, max_seq=64), so.OracleModel(cfg, w, max_seq=64)
    m1.prefill(prompt)
    m2.prefill(prompt)
    r1 = m1.decode(7, 24, True, zero, want_mask=True)
    r2 = m2.decode(7, 24, False)
    assert r1.mask.all()
    np.testing.assert_array_equal(r1.logits, r2.logits)


def test_cats_threshold_recipe(tiny):
    """Reading D3': t(rho) is the (1-rho) quantile of |SiLU(Z)|, Z~N(0,1).  Pinned by Monte Carlo and by
    calibration on the oracle's own dense-prefill gate activations (CATS-style, calibration prompts):
    the measured per-layer quantile is within sampling error of t(rho)."""
    rng = np.random.default_rng(0)
    z = rng.standard_normal(4_000_000)
    absa = np.abs(z / (1 + np.exp(-z)))
    for rho in (0.3, 0.5, 0.7):
        t = synth.cats_threshold(rho)
        assert abs(np.mean(absa >= t) - rho) < 1e-3
    assert synth.cats_threshold(1.0) == 0.0
    cfg, w = tiny
    m = so.OracleModel(cfg, w, max_seq=64)
    gates = [m.forward_row(int(tok), i, want_gate=True).gate for i, tok in enumerate(synth.calib_prompt(cfg, 0, 48))]
    acts = np.abs(np.stack(gates))  # [P, L, ffn]
    t = synth.layer_thresholds(cfg, 0.5)
    for l in range(cfg.n_layers):
        s = np.sort(acts[:, l, :].ravel())
        t_cal = s[int(np.floor(0.5 * s.size))]
        assert abs(t_cal - t[l]) < 0.03, (l, t_cal, t[l])
    # with the per-neuron gains: Monte Carlo of the mixture law
    k = synth.row_gain_k(1000 + 7, cfg.ffn_dim)
    gains = synth.GAIN_TABLE[k.astype(int) + 24].astype(np.float64)
    g = rng.standard_normal((400, gains.size)) * gains
    a = np.abs(g / (1 + np.exp(-g)))
    assert abs(np.mean(a >= synth.cats_threshold(0.5, gains)) - 0.5) < 5e-3


# ------------------------------------------------------------------ Sirius loop
def test_acceptance_threshold_zero_accepts_everything(tiny):
    """north_star / SPEC S:269: r = 0 accepts every sparse token: every kernel advances gamma."""
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.1)
    m = so.OracleModel(cfg, w, max_seq=128)
    res = so.generate(m, synth.eval_prompt(cfg, 4, 32), 24, 4, 0.0, thr)
    assert all(a == 4 for a in res.advances)


def test_exact_argmax_reproduces_dense_greedy(tiny):
    """north_star / SPEC S:456: with exact-argmax acceptance the Sirius output equals dense greedy
    decode token for token (lossless), while the sparse model alone diverges."""
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.1)
    prompt = synth.eval_prompt(cfg, 5, 32)
    dense = so.greedy_decode(so.OracleModel(cfg, w, max_seq=128), prompt, 40)
    sparse = so.greedy_decode(so.OracleModel(cfg, w, max_seq=128), prompt, 40, True, thr)
    m = so.OracleModel(cfg, w, max_seq=160)
    res = so.generate(m, prompt, 40, 4, 0.0, thr, accept_mode=so.ACCEPT_EXACT_ARGMAX)
    assert res.tokens == dense
    assert sparse != dense
    assert any(a < 4 for a in res.advances)  # some drafts were rejected and corrected


def test_accept_scan_brute_force_and_monotone():
    """accept_scan is a linear scan (Alg. 1 lines 12-16); the accepted length is non-increasing in r
    (SPEC S:300)."""
    rng = np.random.default_rng(1)
    for trial in range(200):
        g = int(rng.integers(1, 9))
        lf = rng.standard_normal((g, 16)) * 3
        toks = [int(t) for t in rng.integers(0, 16, g)]
        prev = g
        for r in (0.0, 0.01, 0.05, 0.1, 0.2, 0.5, 1.0):
            j, q = so.accept_scan(lf, toks, r)
            p = np.exp(lf - lf.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            ref = next((i for i in range(g - 1) if p[i, toks[i + 1]] < r), g - 1)
            assert j == ref and j <= prev
            prev = j
            np.testing.assert_allclose(q[:g - 1], [p[i, toks[i + 1]] for i in range(g - 1)], rtol=1e-12)


def test_generate_accounting(tiny):
    """Accounting identities: 1 <= advance <= gamma; committed tokens = sum of advances
    (minus the final kernel's truncated surplus); AAL <= gamma."""
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.1)
    m = so.OracleModel(cfg, w, max_seq=160)
    res = so.generate(m, synth.eval_prompt(cfg, 6, 32), 32, 6, 0.6, thr)
    adv = res.advances
    assert all(1 <= a <= 6 for a in adv)
    assert 1 + sum(adv[:-1]) < 32 <= 1 + sum(adv)
    assert len(res.tokens) == 32
    for k in res.kernels:
        assert k.n_active.shape == (5, cfg.n_layers)


# ------------------------------------------------------------------ paper arithmetic
def test_table2_effective_density_reproduces_paper():
    """Eq. 3 against Table 2's printed triples.  35 of 36 rows
    agree within 1e-3 (the paper truncates to 3 decimals); row PAPER.md:397 (HumanEval CSparse
    Llama-3-8B, 15.10/16 -> printed 0.691, formula 0.712) is inconsistent in the paper itself
    (reading D24)."""
    rows = [r for r in csv.reader(l for l in open(os.path.join(GOLDEN, "table2_effective_density.csv"))
                                  if not l.startswith("#"))]
    assert len(rows) == 36
    bad = []
    for line, task, sp, model, dens, aal, per, printed in rows:
        v = so.effective_density(int(per), float(dens), float(aal))
        if abs(v - float(printed)) > 1e-3:
            bad.append(int(line))
    assert bad == [397]


def test_paper_worked_numbers():
    g = json.load(open(os.path.join(GOLDEN, "paper_arithmetic.json")))
    for key in ("apu_sec52_kernel16", "apu_sec52_kernel10", "apu_70b_offload"):
        e = g[key]
        v = so.effective_density(e["n_sparse"] + 1, e["density"], e["aal"])
        # printed to 2-3 decimals, truncated (0.7852 -> "0.78"): agree to within one printed unit
        unit = 10.0 ** -len(str(e["printed"]).split(".")[1])
        assert abs(v - e["printed"]) < unit, key
        assert abs(so.apu(e["n_sparse"], e["density"], 1.0, e["aal"]) - v) < 1e-15
    e = g["sd_aal_gamma16"]
    aal = so.sd_expected_aal(e["alpha"], e["gamma"])
    assert abs(aal - e["aal_printed"]) < 5e-3
    assert abs((e["gamma"] * e["density"] + 1) / aal - e["apu_printed"]) < 5e-3
    e = g["sd_best_gamma"]
    apus = {gm: (gm * e["density"] + 1) / so.sd_expected_aal(e["alpha"], gm) for gm in range(1, 33)}
    best = min(apus, key=apus.get)
    assert best == e["best_gamma"] and abs(apus[best] - e["apu_printed"]) < 5e-3
    c8 = so.param_counts(synth.LLAMA3_8B)
    assert abs(c8["mlp"] / c8["total"] - g["mlp_fraction_8b"]["printed"]) < 0.01
    c70 = so.param_counts(synth.LLAMA3_70B)
    assert abs(c70["mlp"] / c70["total"] - g["mlp_fraction_70b"]["printed"]) < 0.01
    assert abs(so.global_density(synth.LLAMA3_8B, 0.5, "fsparse") - g["fsparse_density_8b"]["printed"]) < 0.01
    assert abs(so.global_density(synth.LLAMA3_8B, 0.5, "csparse") - g["csparse_density_8b"]["printed"]) < 0.01
    assert abs(so.global_density(synth.LLAMA3_70B, 0.5, "csparse") - g["csparse_apu_70b"]["printed"]) < 0.01


def test_top2_margin():
    assert so.top2_margin(np.array([1.0, 3.0, 2.5])) == 0.5
    assert so.top2_margin(np.array([3.0, 1.0, 3.0])) == 0.0
