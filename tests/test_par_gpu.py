"""Fused peer all-reduce of the tensor-parallel decode step (SURVEY.md §8(e) phase 2; include/sirius.h
sirius_par_enable; csrc/peer_ar.cuh) on one GPU.

One GPU cannot host ranks whose kernels wait on one another (B200_PROFILING.md), so the ranks are
emulated in one context: every emulated rank's producer kernel (O-proj GEMV, CATS FFN, LM head)
pushes as on a real rank, and the wait + rank-order reduction that a real rank's last CTA runs
right after its push (PeerAr.fused) runs, for each emulated rank, in par_reduce_kernel once all of
them have pushed — the same device code (csrc/peer_ar.cuh), so the pushes, the slot / flag
addressing, the sequence numbers, the parities and the reduction order are exercised as on a real
TP group.  The fused form itself (push, wait and reduce in the producer's last CTA) runs on one GPU
in loopback (every peer is the rank's own buffer).

  * bitwise: with the deterministic FFN reduction, the fused path reproduces the in-order-sum
    emulation (the NCCL stand-in) bit for bit — tokens, logits, active counts, gate activations —
    across decode steps interleaved with correct_kernel / kv_rewrite (whose collectives are not
    fused: the sequence numbers must survive them);
  * oracle: the whole Sirius loop free-running at 8B-2L shapes, TP 2, fused path with the default
    atomic FFN, token-exact against the TP-1 oracle;
  * loopback stub (the per-rank timing proxy, fused form): runs, finite, no device error;
  * ABI errors.
The real multi-process path (CUDA IPC handles) is tests/test_tp_nccl_gpu.py (>= 2 GPUs).
"""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def i32(x):
    return torch.tensor(np.asarray(x, dtype=np.int32), device="cuda")


def make_ctx(cfg, w, thr, tp, max_seq=256, max_gamma=16):
    from paper_2409_03856_b200 import sirius as S
    return S.Sirius(cfg, w, thr, batch=1, max_seq=max_seq, max_gamma=max_gamma, tp_size=tp)


def script(ctx, cfg, prompt, steps=10, gamma=4):
    """prefill -> decode steps (sparse, one dense) -> correct_kernel + kv_rewrite -> more decode
    steps; returns every output of every call (host arrays)."""
    from paper_2409_03856_b200 import sirius as S
    L, F, V = cfg.n_layers, cfg.ffn_dim, cfg.vocab
    outs = []
    first = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], first)
    tok, T = int(first.item()), len(prompt)
    drafts = [tok]
    for i in range(steps):
        if i == gamma:  # verify the first gamma drafts, commit, continue after the accepted prefix
            na = torch.zeros(1, dtype=torch.int32, device="cuda")
            nx = torch.zeros(1, dtype=torch.int32, device="cuda")
            q = torch.zeros((1, gamma), dtype=torch.float32, device="cuda")
            ctx.correct_kernel(i32([drafts[:gamma]]), i32([len(prompt)]), gamma, 0.3, 0, na, nx, q, None)
            ctx.kv_rewrite(i32([len(prompt)]), na + 1)
            torch.cuda.synchronize()
            outs.append(("verify", na.cpu().numpy(), nx.cpu().numpy(), q.cpu().numpy()))
            T = len(prompt) + int(na.item()) + 1
            tok = int(nx.item())
        to = torch.zeros(1, dtype=torch.int32, device="cuda")
        lo = torch.zeros((1, V), dtype=torch.float32, device="cuda")
        na = torch.zeros((1, L), dtype=torch.int32, device="cuda")
        ga = torch.zeros((1, L, F), dtype=torch.float32, device="cuda")
        flags = S.SIRIUS_DENSE if i == 2 else 0
        ctx.sparse_decode_step(i32([tok]), i32([T]), flags, to, lo, na, ga)
        torch.cuda.synchronize()
        outs.append(("decode", to.cpu().numpy(), lo.cpu().numpy(), na.cpu().numpy(), ga.cpu().numpy()))
        tok, T = int(to.item()), T + 1
        drafts.append(tok)
    return outs


@pytest.fixture(scope="module")
def l2():
    cfg = synth.LLAMA3_8B.with_layers(2)
    return cfg, synth.host_weights(cfg)


@pytest.mark.parametrize("model,tp", [("tiny", 2), ("8b2l", 2), ("8b2l", 8)])
def test_par_emulated_bitwise_equals_inorder_sum(monkeypatch, model, tp):
    from synth import gpu as sg
    monkeypatch.setenv("SIRIUS_FFN_ATOMIC", "0")  # deterministic FFN: both runs bitwise reproducible
    cfg = synth.TINY if model == "tiny" else synth.LLAMA3_8B.with_layers(2)
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 3, 41)
    shards = [sg.device_weights(cfg, tp, r) for r in range(tp)]
    ref_ctx = make_ctx(cfg, shards, thr, tp)
    ref = script(ref_ctx, cfg, prompt)
    ctx = make_ctx(cfg, shards, thr, tp)
    ctx.sirius_par_enable(None)
    got = script(ctx, cfg, prompt)
    assert len(got) == len(ref)
    for a, b in zip(got, ref):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            np.testing.assert_array_equal(x, y)

    # the peer all-reduce really ran: per decode step, instead of 2 in-order sums per layer and one
    # argmax_finalize, one par_reduce per emulated rank at each of the 2 L + 1 sync points
    def step_launches(c):
        to = torch.zeros(1, dtype=torch.int32, device="cuda")
        n0 = c.launches()
        c.sparse_decode_step(i32([1]), i32([len(prompt) + 20]), 0, to)
        torch.cuda.synchronize()
        return c.launches() - n0
    assert step_launches(ctx) - step_launches(ref_ctx) == (2 * cfg.n_layers + 1) * (tp - 1)


def test_par_emulated_tp2_free_running_token_exact(l2):
    """Sirius free-running at 8B-2L shapes, TP 2 emulated with the fused all-reduce and the default
    (atomic) FFN: tokens and per-kernel advances identical to the TP-1 oracle (prompt chosen free of
    ambiguity events, as in test_parity_8b_gpu.test_8b2l_free_running_token_exact)."""
    from paper_2409_03856_b200 import driver
    from synth import gpu as sg
    from test_parity_8b_gpu import GAMMA, ambiguity_events
    cfg, wh = l2
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 9, 128)
    ref = so.generate(so.OracleModel(cfg, wh, max_seq=256, max_gamma=GAMMA), prompt, 48, GAMMA, 0.3, thr)
    assert ambiguity_events(ref, 0.3) == 0
    ctx = make_ctx(cfg, [sg.device_weights(cfg, 2, r) for r in range(2)], thr, 2)
    ctx.sirius_par_enable(None)
    out = driver.Driver(ctx).sirius([prompt], 48, GAMMA, 0.3)
    assert out.tokens[0] == ref.tokens
    assert out.advances(0) == ref.advances[:len(out.kernels)]


def test_par_loopback_stub_runs(monkeypatch):
    """SIRIUS_DEBUG_STUB_COMM + sirius_par_enable: one rank's TP-8 shard with every push looped back
    into its own buffer (the per-rank timing proxy of tools/tp_proxy.py): runs, no device error."""
    from synth import gpu as sg
    monkeypatch.setenv("SIRIUS_DEBUG_STUB_COMM", "1")
    cfg = synth.LLAMA3_8B.with_layers(2)
    thr = synth.layer_thresholds(cfg, 0.5)
    from paper_2409_03856_b200 import sirius as S
    # stub contexts take a dummy communicator handle (never used: every collective is skipped)
    ctx = S.Sirius(cfg, sg.device_weights(cfg, 8, 0), thr, batch=1, max_seq=256, max_gamma=16, tp_size=8,
                   tp_rank=0, nccl_comm=1)
    ctx.sirius_par_enable(None)
    outs = script(ctx, cfg, synth.eval_prompt(cfg, 2, 30), steps=6)
    for o in outs:
        if o[0] == "decode":
            assert np.isfinite(o[2]).all()


def test_par_abi_errors():
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    cfg = synth.TINY
    thr = synth.layer_thresholds(cfg, 0.5)
    one = make_ctx(cfg, sg.device_weights(cfg), thr, 1)
    with pytest.raises(S.SiriusError) as e:
        one.sirius_par_enable(None)
    assert e.value.status == -6  # UNSUPPORTED: tp_size 1
    emu = make_ctx(cfg, [sg.device_weights(cfg, 2, r) for r in range(2)], thr, 2)
    with pytest.raises(S.SiriusError) as e:
        emu.sirius_par_export()
    assert e.value.status == -3  # STATE: nothing to export from an emulated group
    with pytest.raises(S.SiriusError) as e:
        emu.sirius_par_enable([b"\0" * S.PAR_HANDLE_BYTES] * 2)
    assert e.value.status == -1  # INVALID_ARG: emulated contexts take no handles


def test_par_emulated_batched_rows_bitwise(monkeypatch):
    """Batch 8 (the tensor-core row path for decode; verify of 8 x 4 rows): the fused all-reduce of the
    row forwards (O / down GEMM epilogues push over peer memory, norm_rows sums) reproduces the in-order
    sums bit for bit, tiny TP 2, deterministic FFN."""
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    monkeypatch.setenv("SIRIUS_FFN_ATOMIC", "0")
    cfg, tp, B, gamma = synth.TINY, 2, 8, 4
    thr = synth.layer_thresholds(cfg, 0.5)
    prompts = [synth.eval_prompt(cfg, 20 + b, 9 + 3 * b) for b in range(B)]
    shards = [sg.device_weights(cfg, tp, r) for r in range(tp)]

    def run(par):
        ctx = S.Sirius(cfg, shards, thr, batch=B, max_seq=128, max_gamma=16, tp_size=tp)
        if par:
            ctx.sirius_par_enable(None)
        first = torch.zeros(B, dtype=torch.int32, device="cuda")
        ctx.sirius_prefill(i32(np.concatenate(prompts)), [len(p) for p in prompts], first)
        T = np.array([len(p) for p in prompts], dtype=np.int32)
        tok = first.clone()
        outs, drafts = [], [first.cpu().numpy()]
        for i in range(gamma - 1):
            to = torch.zeros(B, dtype=torch.int32, device="cuda")
            lo = torch.zeros((B, cfg.vocab), dtype=torch.float32, device="cuda")
            ctx.sparse_decode_step(tok, i32(T + i), 0, to, lo)
            torch.cuda.synchronize()
            outs += [to.cpu().numpy(), lo.cpu().numpy()]
            drafts.append(to.cpu().numpy())
            tok = to
        kt = np.stack(drafts, axis=1).astype(np.int32)  # [B, gamma]: pending, d_1 .. d_{gamma-1}
        na = torch.zeros(B, dtype=torch.int32, device="cuda")
        nx = torch.zeros(B, dtype=torch.int32, device="cuda")
        q = torch.zeros((B, gamma), dtype=torch.float32, device="cuda")
        lo = torch.zeros((B, gamma, cfg.vocab), dtype=torch.float32, device="cuda")
        ctx.correct_kernel(i32(kt), i32(T), gamma, 0.3, 0, na, nx, q, lo)
        torch.cuda.synchronize()
        outs += [na.cpu().numpy(), nx.cpu().numpy(), q.cpu().numpy(), lo.cpu().numpy()]
        return outs

    ref, got = run(False), run(True)
    for x, y in zip(got, ref):
        np.testing.assert_array_equal(x, y)


def test_par_missing_peer_times_out_to_nccl_error(monkeypatch):
    """A rank that never publishes (emulated: rank 0's sync-point counter skewed by 2, so its waits
    expect a sequence number nobody writes): the wait gives up after SIRIUS_PAR_TIMEOUT_MS, every
    later wait gives up at once, and the next call returns SIRIUS_ERR_NCCL (sticky)."""
    from paper_2409_03856_b200 import sirius as S
    from synth import gpu as sg
    monkeypatch.setenv("SIRIUS_PAR_TIMEOUT_MS", "200")
    cfg = synth.TINY
    thr = synth.layer_thresholds(cfg, 0.5)
    ctx = make_ctx(cfg, [sg.device_weights(cfg, 2, r) for r in range(2)], thr, 2)
    ctx.graphs(False)
    ctx.sirius_par_enable(None)
    prompt = synth.eval_prompt(cfg, 1, 20)
    first = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sirius_prefill(i32(prompt), [len(prompt)], first)
    to = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.sparse_decode_step(first, i32([len(prompt)]), 0, to)
    torch.cuda.synchronize()
    assert ctx.lib.sirius_debug_par_skew(ctx.h, 0, 2) == 0
    import time
    t0 = time.time()
    ctx.sparse_decode_step(to, i32([len(prompt) + 1]), 0, first)
    torch.cuda.synchronize()
    assert time.time() - t0 < 5.0  # one timeout, not one per sync point
    with pytest.raises(S.SiriusError) as e:
        ctx.sparse_decode_step(first, i32([len(prompt) + 2]), 0, to)
    assert e.value.status == -5  # SIRIUS_ERR_NCCL
