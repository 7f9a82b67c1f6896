"""GPU parity of sampled decoding (reading D31): with
sirius_set_sampling(0.6, seed) the drafted and the interleaved / bonus tokens are drawn by inverse CDF
with the position-keyed counter-based uniform; the free-running Sirius loop must equal the oracle's
(so.generate(temperature=0.6, seed=...)) token for token when no draw lies within float error of a
CDF boundary (the oracle records each drafting row's distance; runs with a near-boundary draw are
rejected as ambiguous, not counted as passes)."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("r,seed", [(0.1, 1), (0.3, 2), (0.0, 3)])
def test_sampled_sirius_token_exact(r, seed):
    from paper_2409_03856_b200 import driver, sirius as S
    from synth import gpu as sg
    cfg = synth.TINY
    wh = synth.host_weights(cfg)
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, seed, 64)
    ref = so.generate(so.OracleModel(cfg, wh, max_seq=256, max_gamma=16), prompt, 32, 4, r, thr, temperature=0.6,
                      seed=seed)
    assert min(float(np.min(k.draft_margin)) for k in ref.kernels) > 1e-5, "ambiguous draw: pick another seed"
    ctx = S.Sirius(cfg, sg.device_weights(cfg), thr, batch=1, max_seq=256, max_gamma=16)
    ctx.sirius_set_sampling(0.6, seed)
    out = driver.Driver(ctx).sirius([prompt], 32, 4, r)
    assert out.tokens[0] == ref.tokens
    assert out.advances(0) == ref.advances[:len(out.kernels)]
    greedy = so.generate(so.OracleModel(cfg, wh, max_seq=256, max_gamma=16), prompt, 32, 4, r, thr)
    assert greedy.tokens != ref.tokens  # sampling changed the run


def test_sampling_errors():
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    cfg = synth.TINY
    ctx = S.Sirius(cfg, sg.device_weights(cfg), synth.layer_thresholds(cfg, 0.5), batch=1, max_seq=64, max_gamma=4)
    with pytest.raises(S.SiriusError) as e:
        ctx.sirius_set_sampling(-1.0)
    assert e.value.status == S.SIRIUS_ERR_INVALID_ARG
