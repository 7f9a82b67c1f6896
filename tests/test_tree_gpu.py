"""GPU parity of tree building + tree verification (reading D29)
through the C ABI (sirius_tree_kernel + kv_rewrite) against the CPU oracle (so.generate(tree_width=W)):
free-running Sirius with trees must produce the oracle's tokens and per-kernel advances; width 1 must
equal the greedy-chain path; the shapes cover the tiny model and the Llama-3-8B layer shapes at the
paper's configuration (kernel 16, width 4: 61 verified rows)."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ctx(cfg, thr, max_gamma=64, max_seq=512):
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    return S.Sirius(cfg, sg.device_weights(cfg), thr, batch=1, max_seq=max_seq, max_gamma=max_gamma)


@pytest.mark.parametrize("r", [0.1, 0.3])
def test_tree_width_one_equals_chain(r):
    from paper_2409_03856_b200 import driver
    cfg = synth.TINY
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 0, 64)
    a = driver.Driver(_ctx(cfg, thr)).sirius([prompt], 32, 4, r)
    b = driver.Driver(_ctx(cfg, thr)).sirius_tree([prompt], 32, 4, r, width=1)
    assert a.tokens == b.tokens and a.advances(0) == b.advances(0)


@pytest.mark.parametrize("width,r,seed", [(2, 0.1, 0), (4, 0.3, 0), (3, 0.3, 5), (4, 0.0, 1)])
def test_tree_free_running_token_exact_tiny(width, r, seed):
    from paper_2409_03856_b200 import driver
    cfg = synth.TINY
    wh = synth.host_weights(cfg)
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, seed, 64)
    gamma = 4
    ref = so.generate(so.OracleModel(cfg, wh, max_seq=512, max_gamma=64), prompt, 32, gamma, r, thr, tree_width=width)
    out = driver.Driver(_ctx(cfg, thr)).sirius_tree([prompt], 32, gamma, r, width=width)
    assert out.tokens[0] == ref.tokens
    assert out.advances(0) == ref.advances[:len(out.kernels)]


def test_tree_8b2l_kernel16_width4():
    """The paper's configuration (kernel 16, tree width 4) at the Llama-3-8B layer shapes: 61 tree rows in
    one tcgen05 verify, ancestor-masked attention over a 128-token prompt; three tree kernels."""
    from paper_2409_03856_b200 import driver
    cfg = synth.LLAMA3_8B_2L
    wh = synth.host_weights(cfg)
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 3, 128)
    ref = so.generate(so.OracleModel(cfg, wh, max_seq=512, max_gamma=64), prompt, 40, 16, 0.3, thr, tree_width=4)
    out = driver.Driver(_ctx(cfg, thr)).sirius_tree([prompt], 40, 16, 0.3, width=4)
    assert out.tokens[0] == ref.tokens
    assert out.advances(0) == ref.advances[:len(out.kernels)]


def test_tree_errors():
    from paper_2409_03856_b200 import sirius as S
    cfg = synth.TINY
    thr = synth.layer_thresholds(cfg, 0.5)
    ctx = _ctx(cfg, thr, max_gamma=16)
    t = torch.zeros(1, dtype=torch.int32, device="cuda")
    p = torch.zeros(16, dtype=torch.int32, device="cuda")
    with pytest.raises(S.SiriusError) as e:  # 1 + 15 * 4 rows > max_gamma 16
        ctx.sirius_tree_kernel(t, t, 16, 4, 3, 0.1, 0, t, t, p)
    assert e.value.status == S.SIRIUS_ERR_CAPACITY
    with pytest.raises(S.SiriusError) as e:
        ctx.sirius_tree_kernel(t, t, 4, 9, 3, 0.1, 0, t, t, p)
    assert e.value.status == S.SIRIUS_ERR_INVALID_ARG
