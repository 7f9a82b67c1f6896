"""Device twin of the synth generator (synth/synth_gpu.cu): fills torch CUDA buffers in HBM."""
from __future__ import annotations

import ctypes
import os

from . import GAIN_STEP, GAIN_TABLE, ModelConfig, TensorSpec, WEIGHT_SEED, shard_blocks, tensor_specs

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _load():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libsynth_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.synth_gpu_fill_bf16.argtypes = [ctypes.c_uint64] * 7 + [ctypes.c_float, ctypes.c_float, ctypes.c_uint64,
                                                                   ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                                                   ctypes.c_void_p]
        lib.synth_gpu_fill_bf16.restype = ctypes.c_int
        lib.synth_gpu_fill_tokens.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                              ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_gpu_fill_tokens.restype = ctypes.c_int
        _lib = lib
    return _lib


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def fill(spec: TensorSpec, row0: int, nrows: int, col0: int, ncols: int, out, seed: int = WEIGHT_SEED) -> None:
    """Write the sub-block of tensor `spec` into the contiguous 2-byte CUDA tensor `out`."""
    assert out.is_cuda and out.is_contiguous() and out.element_size() == 2 and out.numel() == nrows * ncols
    r = _load().synth_gpu_fill_bf16(seed, spec.tensor_id, spec.cols, row0, nrows, col0, ncols, spec.scale,
                                    spec.offset, spec.gain_id, GAIN_STEP, GAIN_TABLE.ctypes.data, out.data_ptr(),
                                    _stream())
    if r != 0:
        raise RuntimeError(f"synth_gpu_fill_bf16: cuda error {r}")


def tokens(seed: int, stream_id: int, n: int, vocab: int, out) -> None:
    r = _load().synth_gpu_fill_tokens(seed, stream_id, n, vocab, out.data_ptr(), _stream())
    if r != 0:
        raise RuntimeError(f"synth_gpu_fill_tokens: cuda error {r}")


def device_weights(cfg: ModelConfig, tp_size: int = 1, tp_rank: int = 0, seed: int = WEIGHT_SEED):
    """All weight tensors of rank tp_rank's shard, generated directly in HBM (torch.bfloat16)."""
    import torch
    out = {}
    for s in tensor_specs(cfg):
        blocks = shard_blocks(cfg, s, tp_size, tp_rank)
        rows = sum(b[1] for b in blocks)
        cols = blocks[0][3]
        t = torch.empty((rows, cols) if s.rows > 1 else (cols,), dtype=torch.bfloat16, device="cuda")
        r = 0
        flat = t.view(-1)
        for (r0, nr, c0, nc) in blocks:
            fill(s, r0, nr, c0, nc, flat[r * nc:(r + nr) * nc], seed)
            r += nr
        out[s.name] = t
    return out
