"""The N > 1 path on CPU: two processes over gloo (127.0.0.1), world size 2.

  * the NCCL bootstrap plumbing of paper_2409_03856_b200/tp.py: rank 0's 128-byte id reaches every
    rank unchanged; max_over_ranks returns the max of the per-rank timings;
  * the tensor-parallel decomposition the CUDA path relies on (reading D1): each
    rank holds ffn/tp neurons of W_gate / W_up / W_down (synth's shard layout, the one
    synth.gpu.device_weights uploads), thresholds ITS OWN shard with the same t_l, and the
    all-reduced sum of the per-rank down-proj partials equals the TP 1 oracle's CATS MLP — the
    global active set is the disjoint union of the per-rank sets.  Likewise the row-sharded
    LM head: the max-reduce of per-rank (value, lowest index) keys is the global argmax.
The per-rank partial below is written out in numpy (fp64) from the definition (PAPER.md:121:
SiLU-gated MLP, threshold on |SiLU(g)|, up / down over the active neurons only).
"""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bf16(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    from oracle import sirius_oracle as so
    from paper_2409_03856_b200 import tp as TP
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ---- bootstrap plumbing
        uid = TP.broadcast_id(rank, lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        assert TP.max_over_ranks(1.5 + rank) == 1.5 + world - 1
        # fused peer all-reduce bootstrap: every rank's IPC handle, in rank order, everywhere
        hs = TP.exchange_handles(bytes([rank]) * 64, 64)
        assert hs == [bytes([r]) * 64 for r in range(world)]

        class FakeCtx:  # the two ABI calls par_bootstrap makes (sirius_par_export / sirius_par_enable)
            got = None

            def sirius_par_export(self):
                return bytes([0xA0 + rank]) * 64

            def sirius_par_enable(self, handles):
                self.got = list(handles)

        fc = FakeCtx()
        TP.par_bootstrap(fc)
        assert fc.got == [bytes([0xA0 + r]) * 64 for r in range(world)]
        TP.barrier()
        # ---- sharded CATS MLP, all-reduced
        cfg = synth.TINY
        full = synth.host_weights(cfg)
        shard = synth.host_weights(cfg, world, rank)
        thr = synth.layer_thresholds(cfg, 0.5)
        rng = np.random.default_rng(7)
        x = rng.standard_normal(cfg.d_model)
        for l in range(cfg.n_layers):
            t = float(np.float32(thr[l]))
            nw = _bf16(shard[f"layers.{l}.ffn_norm"])
            h2 = x / np.sqrt(np.mean(x * x) + cfg.rms_eps) * nw
            g = _bf16(shard[f"layers.{l}.w_gate"]) @ h2
            a = g / (1.0 + np.exp(-g))
            act = np.abs(a) >= t
            u = _bf16(shard[f"layers.{l}.w_up"][act]) @ h2
            y = (a[act] * u) @ _bf16(shard[f"layers.{l}.w_down"][act])
            yt = torch.tensor(y)
            dist.all_reduce(yt)
            cnt = torch.tensor([int(act.sum())])
            dist.all_reduce(cnt)
            om = so.OracleModel(cfg, full, max_seq=8, max_gamma=2, threads=1)
            x_ref, _, mask, n_ref = om.mlp(l, x, True, t)
            assert int(cnt.item()) == n_ref
            np.testing.assert_allclose(x + yt.numpy(), x_ref, rtol=1e-12, atol=1e-12)
            # this rank's active set is exactly its slice of the global one
            F = cfg.ffn_dim // world
            assert np.array_equal(act, mask[rank * F:(rank + 1) * F].astype(bool))
        # ---- vocab-parallel head: max-reduce of packed (value, lowest index) keys
        hf = rng.standard_normal(cfg.d_model)
        logits = _bf16(shard["lm_head"]) @ hf
        V = cfg.vocab // world
        i = int(np.argmax(logits))
        key = torch.tensor([float(logits[i]), -float(rank * V + i)], dtype=torch.float64)
        keys = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(keys, key)
        best = max(keys, key=lambda k: (float(k[0]), float(k[1])))
        ref = _bf16(full["lm_head"]) @ hf
        assert int(-best[1].item()) == so.argmax_lowest(ref)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_tp2_gloo_bootstrap_and_sharded_cats_mlp():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
    assert all(p.exitcode == 0 for p in ps)
