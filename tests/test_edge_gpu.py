"""Edge cases of the C ABI on the GPU (tiny config): the degenerate cases of the method and the
documented error behaviour of include/sirius.h.

  * gamma = 1: the correction kernel verifies only the pending token — no draft to accept,
    n_accept = 0 and the next token is the full model's argmax of that row (Alg. 1 with kernel size 1);
  * no neuron active (t_l above every |a|): the CATS FFN contributes exactly nothing — the oracle with
    the same thresholds is the reference (PAPER.md:121 applied at density 0);
  * gamma > max_gamma -> SIRIUS_ERR_CAPACITY, gamma < 1 / NULL buffers -> SIRIUS_ERR_INVALID_ARG,
    a decode position outside [0, max_seq) -> sticky device-side capacity error reported by the next
    call, kv_rewrite with n_rows outside [1, gamma] -> likewise.
"""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ABS, REL = 2e-2, 1e-2


def i32(x):
    return torch.tensor(np.asarray(x, dtype=np.int32), device="cuda")


@pytest.fixture(scope="module")
def tiny():
    from synth import gpu as sg
    cfg = synth.TINY
    return cfg, synth.host_weights(cfg), sg.device_weights(cfg)


def make_ctx(cfg, wd, thr, max_seq=128, max_gamma=8):
    from paper_2409_03856_b200 import sirius as S
    return S.Sirius(cfg, wd, thr, batch=1, max_seq=max_seq, max_gamma=max_gamma)


def test_gamma_one_is_a_dense_step(tiny):
    cfg, wh, wd = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 11, 30)
    om = so.OracleModel(cfg, wh, max_seq=128, max_gamma=8)
    first = so.argmax_lowest(om.prefill_last(prompt))
    ctx = make_ctx(cfg, wd, thr)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], f)
    lf = om.verify([first], len(prompt))
    na, nx = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda")
    q = torch.zeros((1, 1), dtype=torch.float32, device="cuda")
    lo = torch.zeros((1, 1, cfg.vocab), dtype=torch.float32, device="cuda")
    ctx.correct_kernel(i32([[first]]), i32([len(prompt)]), 1, 0.5, 0, na, nx, q, lo)
    torch.cuda.synchronize()
    assert int(na.item()) == 0
    err = np.abs(lo.cpu().numpy()[0, 0] - lf[0])
    assert np.all(err <= ABS + REL * np.abs(lf[0]))
    s = np.sort(lf[0])
    if s[-1] - s[-2] > 2 * err.max():
        assert int(nx.item()) == so.argmax_lowest(lf[0])
    # q of the last (bonus) row is the probability of its argmax
    p = np.exp(lf[0] - lf[0].max())
    np.testing.assert_allclose(float(q.item()), p.max() / p.sum(), rtol=1e-3)


def test_no_active_neuron(tiny):
    """Thresholds above every |SiLU(g)|: the sparse model's FFN output is exactly zero."""
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd = tiny
    thr = np.full(cfg.n_layers, 1e30, dtype=np.float32)
    prompt = synth.eval_prompt(cfg, 12, 20)
    om = so.OracleModel(cfg, wh, max_seq=128, max_gamma=8)
    tok = so.argmax_lowest(om.prefill_last(prompt))
    ref = om.decode(tok, len(prompt), True, thr, want_mask=True)
    assert ref.mask.sum() == 0
    ctx = make_ctx(cfg, wd, thr)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], f)
    to = torch.zeros(1, dtype=torch.int32, device="cuda")
    lo = torch.zeros((1, cfg.vocab), dtype=torch.float32, device="cuda")
    na = torch.zeros((1, cfg.n_layers), dtype=torch.int32, device="cuda")
    ctx.sparse_decode_step(i32([tok]), i32([len(prompt)]), 0, to, lo, na)
    torch.cuda.synchronize()
    assert np.all(na.cpu().numpy() == 0)
    err = np.abs(lo.cpu().numpy()[0] - ref.logits)
    assert np.all(err <= ABS + REL * np.abs(ref.logits))


def test_error_behaviour(tiny):
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 13, 16)
    ctx = make_ctx(cfg, wd, thr, max_seq=64, max_gamma=4)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], f)
    na, nx = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda")
    kt = i32([[int(f.item())] * 8])
    with pytest.raises(S.SiriusError) as e:  # gamma > max_gamma
        ctx.correct_kernel(kt, i32([16]), 8, 0.1, 0, na, nx)
    assert e.value.status == S.SIRIUS_ERR_CAPACITY
    with pytest.raises(S.SiriusError) as e:  # gamma < 1
        ctx.correct_kernel(kt, i32([16]), 0, 0.1, 0, na, nx)
    assert e.value.status == S.SIRIUS_ERR_INVALID_ARG
    lib = S.load()  # NULL token buffer
    assert lib.sparse_decode_step(ctx.h, None, i32([16]).data_ptr(), 0, nx.data_ptr(), None, None, None) == \
        S.SIRIUS_ERR_INVALID_ARG
    # a decode position outside [0, max_seq): suppressed on the device, reported by a later call
    # (once the stream has run the call that set it)
    ctx.sparse_decode_step(i32([int(f.item())]), i32([64]), 0, nx)
    torch.cuda.synchronize()
    with pytest.raises(S.SiriusError) as e:
        ctx.correct_kernel(i32([[int(f.item())] * 2]), i32([16]), 2, 0.1, 0, na, nx)
    assert e.value.status == S.SIRIUS_ERR_CAPACITY
    with pytest.raises(S.SiriusError) as e:  # sticky
        ctx.sparse_decode_step(i32([int(f.item())]), i32([17]), 0, nx)
    assert e.value.status == S.SIRIUS_ERR_CAPACITY


def test_decode_capacity_error_reported_by_next_decode(tiny):
    """A greedy-only loop (no correct_kernel in between) still sees a device-side capacity error: the
    decode step mirrors the device error word, so the NEXT decode call returns CAPACITY."""
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 14, 16)
    ctx = make_ctx(cfg, wd, thr, max_seq=64, max_gamma=4)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], f)
    nx = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sparse_decode_step(i32([int(f.item())]), i32([64]), 0, nx)  # pos == max_seq: suppressed
    torch.cuda.synchronize()
    with pytest.raises(S.SiriusError) as e:
        ctx.sparse_decode_step(i32([int(f.item())]), i32([17]), 0, nx)
    assert e.value.status == S.SIRIUS_ERR_CAPACITY


@pytest.mark.parametrize("lens", [[1, 9, 1, 33, 2, 1, 17, 5], [257, 1, 300, 3, 260, 1, 4, 258]])
def test_batch8_prefill_single_row_chunks(tiny, lens):
    """Batch 8 (the batched decode row path) with prompts whose last prefill chunk is ONE row (length
    1, or 257 = 256 + 1): that chunk is a prefill of one sequence, not a batched decode step — every
    sequence's first token, its cache and the next decode row match the oracle."""
    from paper_2409_03856_b200 import sirius as S
    cfg, wh, wd = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompts = [synth.eval_prompt(cfg, 40 + b, n) for b, n in enumerate(lens)]
    ctx = S.Sirius(cfg, wd, thr, batch=8, max_seq=384, max_gamma=8)
    f = torch.zeros(8, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(np.concatenate(prompts)), lens, f)
    torch.cuda.synchronize()
    oms, toks = [], []
    for b, p in enumerate(prompts):
        om = so.OracleModel(cfg, wh, max_seq=384, max_gamma=8)
        last = om.prefill_last(p)
        s = np.sort(last)
        if s[-1] - s[-2] > 0.1:
            assert int(f[b].item()) == so.argmax_lowest(last), b
        oms.append(om)
        toks.append(so.argmax_lowest(last))
    to = torch.zeros(8, dtype=torch.int32, device="cuda")
    lo = torch.zeros((8, cfg.vocab), dtype=torch.float32, device="cuda")
    ctx.sparse_decode_step(i32(toks), i32(lens), S.SIRIUS_DENSE, to, lo)
    torch.cuda.synchronize()
    for b in range(8):
        ref = oms[b].decode(toks[b], lens[b], False)
        err = np.abs(lo.cpu().numpy()[b] - ref.logits)
        assert np.all(err <= ABS + REL * np.abs(ref.logits)), (b, float(err.max()))


def _tie_models(tiny, src_offset):
    """Copy the LM-head row of the dense argmax token i of a decode row into row c = i + src_offset
    (same 128-row tile): logits l_i == l_c exactly on both sides."""
    cfg, wh, wd = tiny
    prompt = synth.eval_prompt(cfg, 21, 30)
    om = so.OracleModel(cfg, wh, max_seq=128, max_gamma=8)
    pend = so.argmax_lowest(om.prefill_last(prompt))
    row = om.decode(pend, len(prompt), False).logits
    i = so.argmax_lowest(row)
    c = i + src_offset
    if c < 0 or c >= cfg.vocab or c // 128 != i // 128:
        c = i - src_offset
    wh2 = dict(wh)
    wh2["lm_head"] = wh["lm_head"].copy()
    wh2["lm_head"][c] = wh["lm_head"][i]
    wd2 = dict(wd)
    wd2["lm_head"] = wd["lm_head"].clone()
    wd2["lm_head"][c] = wd["lm_head"][i]
    om2 = so.OracleModel(cfg, wh2, max_seq=128, max_gamma=8)
    om2.prefill_last(prompt)
    ref = om2.decode(pend, len(prompt), False).logits
    assert ref[i] == ref[c] and ref[i] == ref.max()
    return cfg, wh2, wd2, prompt, pend, min(i, c), max(i, c)


@pytest.mark.parametrize("src_offset", [1, -1])
def test_forced_tie_lowest_index(tiny, src_offset):
    """Reading D13 (lowest token id on exact ties) on both GPU paths: two identical LM-head rows give
    an exact logit tie; the decode argmax (GEMV + packed-key atomics), the verify argmax (tcgen05
    GEMM + accept kernel) and the EXACT_ARGMAX accept rule must all pick the LOWER index."""
    from paper_2409_03856_b200 import sirius as S
    cfg, wh2, wd2, prompt, pend, lo_id, hi_id = _tie_models(tiny, src_offset)
    T = len(prompt)
    thr = synth.layer_thresholds(cfg, 0.5)
    ctx = make_ctx(cfg, wd2, thr)
    f = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [T], f)
    to = torch.zeros(1, dtype=torch.int32, device="cuda")
    lo = torch.zeros((1, cfg.vocab), dtype=torch.float32, device="cuda")
    ctx.sparse_decode_step(i32([pend]), i32([T]), S.SIRIUS_DENSE, to, lo)
    torch.cuda.synchronize()
    lg = lo.cpu().numpy()[0]
    assert lg[lo_id] == lg[hi_id] and lg[lo_id] == lg.max()  # exact tie on the GPU too
    assert int(to.item()) == lo_id
    na, nx = torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda")
    q = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    lv = torch.zeros((1, 2, cfg.vocab), dtype=torch.float32, device="cuda")
    for draft, j_expect in ((hi_id, 0), (lo_id, 1)):  # EXACT_ARGMAX: only the lowest tied id is "the argmax"
        ctx.correct_kernel(i32([[pend, draft]]), i32([T]), 2, 0.0, S.ACCEPT_EXACT_ARGMAX, na, nx, q, lv)
        torch.cuda.synchronize()
        v0 = lv.cpu().numpy()[0, 0]
        assert v0[lo_id] == v0[hi_id] and v0[lo_id] == v0.max()
        assert int(na.item()) == j_expect
        if j_expect == 0:
            assert int(nx.item()) == lo_id  # interleaved token = lowest-index argmax of row 0
    ctx.correct_kernel(i32([[pend]]), i32([T]), 1, 0.5, 0, na, nx, q[:, :1].contiguous())
    torch.cuda.synchronize()
    assert int(na.item()) == 0 and int(nx.item()) == lo_id
