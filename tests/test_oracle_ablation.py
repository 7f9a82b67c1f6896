"""Pins for the oracle's component ablation (Table 4; §5.3 PAPER.md:524-525;
reading D27) and the rejection-position statistic.  CPU only."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

MODES = {  # Table 4 rows: (rewrite, interleave, rollback)
    "interleave": (False, True, False),
    "kv_rewrite": (True, False, False),
    "kv_rewrite+interleave": (True, True, False),
    "rollback+interleave": (False, True, True),
    "sirius": (True, True, True),
}


def run(tiny, mode, r, n=24, gamma=4, seed=2):
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.1)
    k, i, rb = MODES[mode]
    m = so.OracleModel(cfg, w, max_seq=160, max_gamma=8)
    return so.generate(m, synth.eval_prompt(cfg, seed, 32), n, gamma, r, thr, rewrite=k, interleave=i, rollback=rb)


def test_advances_by_mode(tiny):
    for mode, (_, _, rb) in MODES.items():
        res = run(tiny, mode, 0.6)
        if rb:
            assert all(1 <= a <= 4 for a in res.advances) and any(a < 4 for a in res.advances)
        else:
            assert all(a == 4 for a in res.advances)
        assert len(res.tokens) == 24


def test_no_rejection_makes_interleave_and_rollback_irrelevant(tiny):
    """r = 0 accepts every draft: interleaving and rollback never act, so the modes coincide pairwise
    (with the same KV policy)."""
    assert run(tiny, "interleave", 0.0).tokens == run(tiny, "rollback+interleave", 0.0).tokens
    assert run(tiny, "kv_rewrite+interleave", 0.0).tokens == run(tiny, "sirius", 0.0).tokens
    assert run(tiny, "kv_rewrite", 0.0).tokens == run(tiny, "sirius", 0.0).tokens


def test_interleave_only_first_kernel_against_dense_prefill(tiny):
    """Interleave-only (no rollback, no rewrite), first kernel: a rejected draft d_{i+1} is replaced by
    the dense model's argmax at position T+i given [prompt, pending, d_1..d_i] — recomputed here by a
    plain dense prefill of that sequence (chunk == sequential); accepted drafts are kept."""
    cfg, w = tiny
    res = run(tiny, "interleave", 0.9, n=4)
    k = res.kernels[0]
    prompt = list(synth.eval_prompt(cfg, 2, 32))
    ref = so.OracleModel(cfg, w, max_seq=64).prefill(prompt + k.tokens)
    P = len(prompt)
    rej = 0
    for i in range(3):
        full_tok = so.argmax_lowest(ref[P + i])
        expect = k.tokens[i + 1] if k.q[i] >= 0.9 else full_tok
        rej += int(k.q[i] < 0.9)
        assert res.tokens[1 + i] == expect
    assert rej > 0


def test_rejection_positions(tiny):
    res = run(tiny, "sirius", 0.6, n=40)
    pos = res.rejection_positions()
    assert pos == [k.j for k in res.kernels if k.j < 3]
    assert all(0 <= p < 3 for p in pos) and len(pos) > 0


def test_rollback_requires_interleave(tiny):
    cfg, w = tiny
    with pytest.raises(AssertionError):
        so.generate(so.OracleModel(cfg, w, max_seq=160), synth.eval_prompt(cfg, 2, 32), 8, 4, 0.5,
                    synth.layer_thresholds(cfg, 0.1), interleave=False, rollback=True)
