"""The seeded input generator (synth/): determinism, the recipe's distribution, shard consistency,
a frozen checksum, and (GPU) bit-equality of the CUDA twin with the C twin."""
import hashlib
import json
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_irwin_hall_range_and_moments():
    z = np.array([synth.irwin_hall(0, 77, i) for i in range(20000)])
    assert z.min() >= -131070 and z.max() <= 131070
    assert abs(z.mean()) < 0.03 * synth.IH_STD
    assert abs(z.std() / synth.IH_STD - 1.0) < 0.02


def test_weights_deterministic_and_scaled():
    cfg = synth.TINY
    specs = {s.name: s for s in synth.tensor_specs(cfg)}
    a = synth.host_shard(cfg, specs["layers.1.w_gate"])
    b = synth.host_shard(cfg, specs["layers.1.w_gate"])
    np.testing.assert_array_equal(a, b)
    f = (a.astype(np.uint32) << 16).view(np.float32)
    # fan-in scaled rows times the per-neuron gain 2^(k/4): row std * sqrt(d) == gain
    k = synth.row_gain_k(specs["layers.1.w_gate"].gain_id, cfg.ffn_dim)
    gains = synth.GAIN_TABLE[k.astype(int) + 24]
    ratio = f.std(axis=1) * np.sqrt(cfg.d_model) / gains
    assert abs(np.median(ratio) - 1.0) < 0.02 and np.all(np.abs(ratio - 1) < 0.25)
    assert 1.0 < np.std(k / 4.0 * np.log(2.0)) / synth.GAIN_SIGMA * 1.0 + 0.2  # log-gain spread ~ sigma
    assert abs(np.std(k / 4.0 * np.log(2.0)) - synth.GAIN_SIGMA) < 0.1
    np.testing.assert_array_equal(synth.host_shard(cfg, specs["layers.1.w_up"]).shape, a.shape)
    n = (synth.host_shard(cfg, specs["final_norm"]).astype(np.uint32) << 16).view(np.float32)
    assert abs(n.mean() - 1.0) < 0.02 and 0.05 < n.std() < 0.15
    c = synth.host_shard(cfg, specs["layers.0.w_gate"])
    assert not np.array_equal(a, c)


def test_shards_are_slices_of_the_full_tensor():
    """TP shards are exactly sub-blocks of the unsharded tensor."""
    cfg = synth.ModelConfig("t", vocab=64, d_model=64, n_layers=1, n_heads=4, n_kv_heads=2, head_dim=16, ffn_dim=96)
    for s in synth.tensor_specs(cfg):
        full = synth.host_shard(cfg, s)
        name = s.name.split(".")[-1]
        for tp in (2,):
            parts = [synth.host_shard(cfg, s, tp, r) for r in range(tp)]
            if name in ("embed", "final_norm", "attn_norm", "ffn_norm"):
                for p in parts:
                    np.testing.assert_array_equal(p, full)
            elif name == "w_o":
                np.testing.assert_array_equal(np.concatenate(parts, axis=1), full)
            elif name == "w_qkv":
                hd, H, KV = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
                q = np.concatenate([p[:H // tp * hd] for p in parts])
                k = np.concatenate([p[H // tp * hd:(H + KV) // tp * hd] for p in parts])
                v = np.concatenate([p[(H + KV) // tp * hd:] for p in parts])
                np.testing.assert_array_equal(np.concatenate([q, k, v]), full)
            else:
                np.testing.assert_array_equal(np.concatenate(parts), full)


def test_frozen_checksum():
    """The generator's output is frozen (tests/golden/synth_checksums.json, written once by
    tests/golden/make_synth_checksums.py, which calls synth/ only)."""
    ref = json.load(open(os.path.join(GOLDEN, "synth_checksums.json")))
    cfg = synth.TINY
    for s in synth.tensor_specs(cfg):
        h = hashlib.sha256(synth.host_shard(cfg, s).tobytes()).hexdigest()
        assert h == ref["tiny"][s.name], s.name
    p = synth.eval_prompt(cfg, 0, 64)
    assert hashlib.sha256(p.tobytes()).hexdigest() == ref["tiny_prompt0_64"]


@pytest.mark.gpu
def test_gpu_generator_bit_equal_to_cpu_generator():
    import torch
    from synth import gpu as synth_gpu
    cfg = synth.LLAMA3_8B
    specs = {s.name: s for s in synth.tensor_specs(cfg)}
    for name, (r0, nr, c0, nc) in [("layers.3.w_gate", (1000, 37, 0, 4096)), ("lm_head", (128000, 256, 0, 4096)),
                                   ("layers.31.w_o", (17, 5, 1024, 512)), ("final_norm", (0, 1, 0, 4096))]:
        s = specs[name]
        cpu = synth.fill_host(s, r0, nr, c0, nc)
        gpu = torch.empty((nr, nc), dtype=torch.int16, device="cuda")
        synth_gpu.fill(s, r0, nr, c0, nc, gpu)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(gpu.cpu().numpy().view(np.uint16), cpu)
    tok = torch.empty(64, dtype=torch.int32, device="cuda")
    synth_gpu.tokens(1, 0, 64, cfg.vocab, tok)
    np.testing.assert_array_equal(tok.cpu().numpy(), synth.prompt_tokens(1, 0, 64, cfg.vocab))
