"""Seeded synthetic inputs shared by the oracle side and the GPU side.

This package holds the *input recipe* only: model shapes, the
counter-based weight/prompt generators (a C twin in ``synth_cpu.c`` and a CUDA
twin in ``synth_gpu.cu``, written independently and cross-checked bit for bit by
``tests/test_synth.py``), and the CATS threshold recipe.  None of the Sirius
method's arithmetic lives here.

Why these gains (SURVEY.md §8(d) "Gains", fixed before any measurement):
  * every projection is fan-in scaled (unit-variance outputs for unit-RMS inputs);
  * the embedding has unit variance;
  * the LM head has gain 5 (logit std ~5), so the full model's next-token
    distribution is peaked enough that the likelihood threshold r=0.1 both
    accepts and rejects (a std-0.02 init gives a flat distribution, AAL = 1);
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
    head_gain: float = 5.0

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
LAYER_NAMES = ("attn_norm", "w_qkv", "w_o", "ffn_norm", "w_gate", "w_up", "w_down")


@dataclass(frozen=True)
class TensorSpec:
    name: str
    tensor_id: int
    rows: int  # full (unsharded) shape
    cols: int
    scale: float  # fp32 multiplier of the Irwin-Hall integer
    offset: float  # fp32 additive offset (1.0 for norm weights)


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
            TensorSpec(f"layers.{l}.w_gate", b + 4, cfg.ffn_dim, d, _f32(1.0 / (math.sqrt(d) * IH_STD)), 0.0),
            TensorSpec(f"layers.{l}.w_up", b + 5, cfg.ffn_dim, d, _f32(1.0 / (math.sqrt(d) * IH_STD)), 0.0),
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
        lib.synth_fill_bf16.argtypes = [ctypes.c_uint64] * 7 + [ctypes.c_float, ctypes.c_float, ctypes.c_void_p,
                                                               ctypes.c_int]
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
                                out.ctypes.data, host_threads())
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
def _silu(z: float) -> float:
    return z / (1.0 + math.exp(-z))


def _phi(z: float) -> float:
    return 0.5 * (1.0 + math.erf(z / math.sqrt(2.0)))


def _solve(f, lo: float, hi: float) -> float:
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(lo) * f(mid) <= 0:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


SILU_NEG_MIN_Z = _solve(lambda z: 1.0 / (1.0 + math.exp(-z)) * (1.0 + z * (1.0 - 1.0 / (1.0 + math.exp(-z)))),
                        -3.0, -0.5)  # argmin of SiLU on z<0 (≈ -1.2785)
SILU_NEG_MIN = -_silu(SILU_NEG_MIN_Z)  # ≈ 0.2785


def abs_silu_cdf(t: float) -> float:
    """P(|SiLU(Z)| <= t) for Z ~ N(0,1)."""
    if t <= 0:
        return 0.0
    zp = _solve(lambda z: _silu(z) - t, 0.0, 50.0)
    p = _phi(zp) - 0.5
    if t >= SILU_NEG_MIN:
        return p + 0.5
    z1 = _solve(lambda z: -_silu(z) - t, -60.0, SILU_NEG_MIN_Z)
    z2 = _solve(lambda z: -_silu(z) - t, SILU_NEG_MIN_Z, 0.0)
    return p + _phi(z1) + (0.5 - _phi(z2))


def cats_threshold(rho: float) -> float:
    """Per-layer CATS threshold t with P(|SiLU(g)| >= t) = rho, under the synthetic init's gate
    pre-activation law g ~ N(0, 1) (unit-RMS h, fan-in-scaled W_gate).  DESIGN.md reading D3'.
    Returned as an fp32 value; both sides receive the same fp32 number."""
    if rho >= 1.0:
        return 0.0
    t = _solve(lambda t: abs_silu_cdf(t) - (1.0 - rho), 1e-9, 30.0)
    return _f32(t)


def layer_thresholds(cfg: ModelConfig, rho) -> np.ndarray:
    """fp32 [n_layers]; rho may be a scalar or a per-layer sequence."""
    if np.isscalar(rho):
        rho = [rho] * cfg.n_layers
    return np.array([cats_threshold(r) for r in rho], dtype=np.float32)
