"""Seeded synthetic inputs shared by the oracle side and the GPU side.

This package holds the *input recipe* only: model shapes, the
counter-based weight/prompt generators (a C twin in ``synth_cpu.c`` and a CUDA
twin in ``synth_gpu.cu``, written independently and cross-checked bit for bit by
``tests/test_synth.py``), and the CATS threshold recipe.  None of the Sirius
method's arithmetic lives here.

Why these gains (SURVEY.md §8(d) "Gains", fixed before any measurement):
  * every projection is fan-in scaled (unit-variance outputs for unit-RMS inputs);
  * the embedding has unit variance;
  * every neuron i of a layer has a gain s_i on its W_gate and W_up rows, log-normal-like
    (s_i = 2^(k_i/4), k_i a rounded Gaussian, sigma_ln = 1.25): the heavy-tailed activation
    magnitudes of trained LLMs that CATS thresholding relies on; with Gaussian
    gates (no gain) 50% thresholding keeps too little of the MLP and the sparse model's drafts are
    rejected almost always (AAL 1.5/16 measured);
  * the LM head has gain 10 (logit std ~10): a next-token distribution about as peaked as the
    paper's, so the likelihood threshold both accepts and rejects; with gain 1.25/head 10 the
    Llama-3-8B shape gives AAL ~15.5/16 at r=0.1 and ~12.7 at r=0.3 (Table 8:
    14.6 and 11.6) — chosen on a GPU sweep (tools/explore_recipe.py) before any timing;
  * RMSNorm weights are 1 + N(0, 0.1^2)-ish (not exactly 1, so a mis-indexed norm
    weight is caught by the parity tests).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace
from typing import Dict, List, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
IH_STD = 65536.0 / math.sqrt(3.0)  # std of (sum of four u16 lanes - 131070) = 37837.23
NORM_STD = 0.1


@dataclass(frozen=True)
class ModelConfig:
    """Llama-style decoder shape (public Llama-3 configs; SURVEY.md §0 'Llama-3 shapes')."""

    name: str
    vocab: int
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    head_gain: float = 10.0

    @property
    def qkv_rows(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def with_layers(self, n: int) -> "ModelConfig":
        return replace(self, n_layers=n, name=f"{self.name}-{n}L")


TINY = ModelConfig("tiny", vocab=512, d_model=256, n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64, ffn_dim=688)
LLAMA3_8B = ModelConfig("llama3-8b", vocab=128256, d_model=4096, n_layers=32, n_heads=32, n_kv_heads=8,
                        head_dim=128, ffn_dim=14336)
LLAMA3_70B = ModelConfig("llama3-70b", vocab=128256, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8,
                         head_dim=128, ffn_dim=28672)
LLAMA3_8B_2L = LLAMA3_8B.with_layers(2)

CONFIGS = {c.name: c for c in (TINY, LLAMA3_8B, LLAMA3_70B, LLAMA3_8B_2L)}

WEIGHT_SEED = 0
GAIN_SIGMA = 1.25  # ln-space std of the per-neuron gate/up gain
GAIN_STEP = int(round(IH_STD * math.log(2.0) / (4.0 * GAIN_SIGMA)))  # IH units per quarter octave (5245)
GAIN_TABLE = np.array([2.0 ** ((j - 24) / 4.0) for j in range(49)], dtype=np.float32)
LAYER_NAMES = ("attn_norm", "w_qkv", "w_o", "ffn_norm", "w_gate", "w_up", "w_down")


@dataclass(frozen=True)
class TensorSpec:
    name: str
    tensor_id: int
    rows: int  # full (unsharded) shape
    cols: int
    scale: float  # fp32 multiplier of the Irwin-Hall integer
    offset: float  # fp32 additive offset (1.0 for norm weights)
    gain_id: int = 0  # != 0: per-row gain 2^(k/4), k from the Irwin-Hall stream `gain_id`


def _f32(x: float) -> float:
    return float(np.float32(x))


def tensor_specs(cfg: ModelConfig) -> List[TensorSpec]:
    """Every weight tensor of the model, full shapes (rows = output features / neurons)."""
    d = cfg.d_model
    norm = dict(scale=_f32(NORM_STD / IH_STD), offset=1.0)
    specs = [
        TensorSpec("embed", 1, cfg.vocab, d, _f32(1.0 / IH_STD), 0.0),
        TensorSpec("final_norm", 2, 1, d, **norm),
        TensorSpec("lm_head", 3, cfg.vocab, d, _f32(cfg.head_gain / (math.sqrt(d) * IH_STD)), 0.0),
    ]
    for l in range(cfg.n_layers):
        b = 1000 + 16 * l
        hd = cfg.head_dim
        specs += [
            TensorSpec(f"layers.{l}.attn_norm", b + 0, 1, d, **norm),
            TensorSpec(f"layers.{l}.w_qkv", b + 1, cfg.qkv_rows, d, _f32(1.0 / (math.sqrt(d) * IH_STD)), 0.0),
            TensorSpec(f"layers.{l}.w_o", b + 2, d, cfg.n_heads * hd,
                       _f32(1.0 / (math.sqrt(cfg.n_heads * hd) * IH_STD)), 0.0),
            TensorSpec(f"layers.{l}.ffn_norm", b + 3, 1, d, **norm),
            TensorSpec(f"layers.{l}.w_gate", b + 4, cfg.ffn_dim, d, _f32(1.0 / (math.sqrt(d) * IH_STD)), 0.0,
                       gain_id=b + 7),
            TensorSpec(f"layers.{l}.w_up", b + 5, cfg.ffn_dim, d, _f32(1.0 / (math.sqrt(d) * IH_STD)), 0.0,
                       gain_id=b + 7),
            # neuron-major W_down: row i is neuron i's d-vector; fan-in of the product is ffn_dim
            TensorSpec(f"layers.{l}.w_down", b + 6, cfg.ffn_dim, d,
                       _f32(1.0 / (math.sqrt(cfg.ffn_dim) * IH_STD)), 0.0),
        ]
    return specs


def shard_blocks(cfg: ModelConfig, spec: TensorSpec, tp_size: int, tp_rank: int) -> List[Tuple[int, int, int, int]]:
    """Sub-blocks (row0, nrows, col0, ncols) of the full tensor that make up rank tp_rank's shard,
    concatenated along rows in the listed order (SURVEY.md §8(e) partitioning)."""
    name = spec.name.split(".")[-1]
    R, C = spec.rows, spec.cols
    if tp_size == 1 or name in ("embed", "final_norm", "attn_norm", "ffn_norm"):
        return [(0, R, 0, C)]
    hd = cfg.head_dim
    if name == "w_qkv":
        hq, hk = cfg.n_heads // tp_size, cfg.n_kv_heads // tp_size
        q0 = tp_rank * hq * hd
        k0 = cfg.n_heads * hd + tp_rank * hk * hd
        v0 = (cfg.n_heads + cfg.n_kv_heads) * hd + tp_rank * hk * hd
        return [(q0, hq * hd, 0, C), (k0, hk * hd, 0, C), (v0, hk * hd, 0, C)]
    if name == "w_o":
        w = C // tp_size
        return [(0, R, tp_rank * w, w)]
    # lm_head, w_gate, w_up, w_down: row-sharded
    r = R // tp_size
    return [(tp_rank * r, r, 0, C)]


# ---------------------------------------------------------------- C generator
_cpu_lib = None


def _load_cpu():
    global _cpu_lib
    if _cpu_lib is None:
        path = os.path.join(_HERE, "libsynth_cpu.so")
        if not os.path.exists(path):
            build_cpu()
        lib = ctypes.CDLL(path)
        lib.synth_fill_bf16.argtypes = [ctypes.c_uint64] * 7 + [ctypes.c_float, ctypes.c_float, ctypes.c_uint64,
                                                               ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                                               ctypes.c_int]
        lib.synth_row_gain_ks.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                          ctypes.c_void_p]
        lib.synth_fill_bf16.restype = None
        lib.synth_fill_tokens.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                          ctypes.c_void_p]
        lib.synth_irwin_hall.argtypes = [ctypes.c_uint64] * 3
        lib.synth_irwin_hall.restype = ctypes.c_int32
        _cpu_lib = lib
    return _cpu_lib


def build_cpu() -> None:
    import subprocess
    src = os.path.join(_HERE, "synth_cpu.c")
    out = os.path.join(_HERE, "libsynth_cpu.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", "-o", out, src])


def irwin_hall(seed: int, tensor_id: int, i: int) -> int:
    return int(_load_cpu().synth_irwin_hall(seed, tensor_id, i))


def host_threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def fill_host(spec: TensorSpec, row0: int, nrows: int, col0: int, ncols: int, seed: int = WEIGHT_SEED) -> np.ndarray:
    """bf16 bit patterns (uint16 [nrows, ncols]) of a sub-block of tensor `spec`."""
    out = np.empty((nrows, ncols), dtype=np.uint16)
    _load_cpu().synth_fill_bf16(seed, spec.tensor_id, spec.cols, row0, nrows, col0, ncols, spec.scale, spec.offset,
                                spec.gain_id, GAIN_STEP, GAIN_TABLE.ctypes.data, out.ctypes.data, host_threads())
    return out


def host_shard(cfg: ModelConfig, spec: TensorSpec, tp_size: int = 1, tp_rank: int = 0,
               seed: int = WEIGHT_SEED) -> np.ndarray:
    blocks = [fill_host(spec, r0, nr, c0, nc, seed) for (r0, nr, c0, nc) in shard_blocks(cfg, spec, tp_size, tp_rank)]
    out = np.concatenate(blocks, axis=0) if len(blocks) > 1 else blocks[0]
    return out.reshape(-1) if spec.rows == 1 else out


def host_weights(cfg: ModelConfig, tp_size: int = 1, tp_rank: int = 0, seed: int = WEIGHT_SEED) -> Dict[str, np.ndarray]:
    """All weights as uint16 bf16 bit arrays, keyed by tensor name."""
    return {s.name: host_shard(cfg, s, tp_size, tp_rank, seed) for s in tensor_specs(cfg)}


def prompt_tokens(seed: int, stream: int, n: int, vocab: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _load_cpu().synth_fill_tokens(seed, stream, n, vocab, out.ctypes.data)
    return out


# seeds: weights 0, calibration prompts 1000+b, eval prompts 1+b
def eval_prompt(cfg: ModelConfig, b: int, n: int) -> np.ndarray:
    return prompt_tokens(1 + b, 0, n, cfg.vocab)


def calib_prompt(cfg: ModelConfig, b: int, n: int) -> np.ndarray:
    return prompt_tokens(1000 + b, 0, n, cfg.vocab)


# ---------------------------------------------------------------- CATS thresholds
def row_gain_k(gain_id: int, n: int, seed: int = WEIGHT_SEED) -> np.ndarray:
    out = np.empty(n, dtype=np.int8)
    _load_cpu().synth_row_gain_ks(seed, gain_id, n, GAIN_STEP, out.ctypes.data)
    return out


def _silu(z: float) -> float:
    return z / (1.0 + math.exp(-z))


def _root(f, lo: float, hi: float) -> float:
    from scipy.optimize import brentq
    return brentq(f, lo, hi, xtol=1e-14, rtol=1e-14, maxiter=500)


SILU_NEG_MIN_Z = _root(lambda z: (1.0 + z * (1.0 - 1.0 / (1.0 + math.exp(-z)))), -3.0, -0.5)  # argmin SiLU (-1.2785)
SILU_NEG_MIN = -_silu(SILU_NEG_MIN_Z)  # 0.2785


def _abs_silu_tail(t: float, sig: np.ndarray) -> np.ndarray:
    """P(|SiLU(X)| >= t) for X ~ N(0, sig^2) (vectorised over sig).  {|SiLU(y)| < t} is
    (z1, zp) minus [.., z2] pieces: SiLU rises on y > 0 to zp, and on y < 0 |SiLU| rises to its
    maximum 0.2785 at y = -1.2785 (z1 < -1.2785 < z2 bound the part above t) then decays."""
    from scipy.special import ndtr
    if t <= 0:
        return np.ones_like(sig)
    zp = _root(lambda y: _silu(y) - t, 0.0, t + 60.0)
    below = ndtr(zp / sig) - 0.5  # 0 <= y < zp
    if t >= SILU_NEG_MIN:
        below = below + 0.5
    else:
        z1 = _root(lambda y: -_silu(y) - t, -80.0, SILU_NEG_MIN_Z)
        z2 = _root(lambda y: -_silu(y) - t, SILU_NEG_MIN_Z, 0.0)
        below = below + ndtr(z1 / sig) + (0.5 - ndtr(z2 / sig))
    return 1.0 - below


def cats_threshold(rho: float, gains=None, var: float = 1.0) -> float:
    """CATS threshold t with mean_i P(|SiLU(g_i)| >= t) = rho under the synthetic init's law of the
    gate pre-activation: g_i ~ N(0, var * s_i^2) (unit-RMS normalised input times the layer's ffn_norm
    weight (var = mean(w^2)), fan-in-scaled W_gate row with gain s_i).  DESIGN.md reading D3'.
    Returned as fp32; both sides receive the same fp32 number."""
    if rho >= 1.0:
        return 0.0
    sig = np.sqrt(var) * (np.ones(1) if gains is None else np.asarray(gains, dtype=np.float64))
    f = lambda t: float(np.mean(_abs_silu_tail(t, sig))) - rho
    return _f32(_root(f, 1e-12, 60.0 * float(sig.max()) + 1.0))


def layer_thresholds(cfg: ModelConfig, rho, seed: int = WEIGHT_SEED) -> np.ndarray:
    """fp32 [n_layers]; rho may be a scalar or a per-layer sequence."""
    if np.isscalar(rho):
        rho = [rho] * cfg.n_layers
    specs = {s.name: s for s in tensor_specs(cfg)}
    out = []
    for l, r in enumerate(rho):
        k = row_gain_k(specs[f"layers.{l}.w_gate"].gain_id, cfg.ffn_dim, seed)
        kv, cnt = np.unique(k, return_counts=True)
        gains = np.repeat(GAIN_TABLE[kv.astype(int) + 24].astype(np.float64), cnt)
        w = (host_shard(cfg, specs[f"layers.{l}.ffn_norm"]).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        # unique gains with multiplicities: mean over neurons == weighted mean over distinct gains
        out.append(cats_threshold(r, gains, float(np.mean(w * w))))
    return np.array(out, dtype=np.float32)


def residual_rows(seed: int, n: int, d: int) -> np.ndarray:
    """Seeded synthetic residual-stream rows (fp32 [n, d]) for kernel-isolated tests of one layer:
    unit-RMS Gaussian rows with a few heavy channels (x8 on 1% of the coordinates), the shape of a
    Llama residual stream.  Handed to both sides as the same array."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    x[:, rng.choice(d, max(1, d // 100), replace=False)] *= 8.0
    x *= rng.uniform(0.5, 3.0, (n, 1))
    return x.astype(np.float32)
