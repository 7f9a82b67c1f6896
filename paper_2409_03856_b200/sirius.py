"""Thin ctypes binding of libsirius (include/sirius.h): argument marshalling only.

Every entry point has the C name: ``sirius_init``, ``sirius_prefill``, ``sparse_decode_step``,
``correct_kernel``, ``kv_rewrite``, ``sirius_destroy``.  Tensors are torch CUDA tensors (torch is
used for device memory and streams only); the library is loaded from this directory and nothing
falls back to the CPU: if the CUDA library or a GPU is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsirius.so")

SIRIUS_OK = 0
SIRIUS_ERR_INVALID_ARG, SIRIUS_ERR_CAPACITY, SIRIUS_ERR_STATE = -1, -2, -3
SIRIUS_ERR_CUDA, SIRIUS_ERR_NCCL, SIRIUS_ERR_UNSUPPORTED = -4, -5, -6
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "CAPACITY", -3: "STATE", -4: "CUDA", -5: "NCCL", -6: "UNSUPPORTED"}
SIRIUS_DENSE = 1
SIRIUS_CSPARSE = 2
SIRIUS_TOPK = 4
ACCEPT_THRESHOLD = 0
ACCEPT_EXACT_ARGMAX = 1
PAR_HANDLE_BYTES = 64  # include/sirius.h SIRIUS_PAR_HANDLE_BYTES (sizeof(cudaIpcMemHandle_t))

# every symbol include/sirius.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ("sirius_init", "sirius_prefill", "sparse_decode_step", "correct_kernel", "kv_rewrite",
               "sirius_verify_row_argmax", "sirius_csparse_enable", "sirius_tree_kernel", "sirius_topk_enable",
               "sirius_set_sampling", "sirius_par_export", "sirius_par_enable", "sirius_par_disable",
               "sirius_destroy",
               "sirius_last_error", "sirius_version")


class SiriusError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sirius status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class SiriusConfig(ctypes.Structure):
    _fields_ = [("vocab", ctypes.c_int32), ("d_model", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("ffn_dim", ctypes.c_int32), ("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float),
                ("batch", ctypes.c_int32), ("max_seq", ctypes.c_int32), ("max_gamma", ctypes.c_int32),
                ("tp_size", ctypes.c_int32), ("tp_rank", ctypes.c_int32)]


_PP = ctypes.POINTER(ctypes.c_void_p)


class SiriusWeights(ctypes.Structure):
    _fields_ = [("embed", ctypes.c_void_p), ("final_norm", ctypes.c_void_p), ("lm_head", ctypes.c_void_p),
                ("attn_norm", _PP), ("w_qkv", _PP), ("w_o", _PP), ("ffn_norm", _PP), ("w_gate", _PP),
                ("w_up", _PP), ("w_down", _PP)]


_lib = None


def load():
    """Load libsirius.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        # SIRIUS_LIB: another build of the same library (A/B timing of kernel variants; tools/)
        path = os.environ.get("SIRIUS_LIB", LIB_PATH)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        P, I, U, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_float
        lib.sirius_init.argtypes = [ctypes.POINTER(SiriusConfig), ctypes.POINTER(SiriusWeights), P, P, P,
                                    ctypes.POINTER(P)]
        lib.sirius_init.restype = I
        lib.sirius_prefill.argtypes = [P, P, P, P]
        lib.sirius_prefill.restype = I
        lib.sparse_decode_step.argtypes = [P, P, P, U, P, P, P, P]
        lib.sparse_decode_step.restype = I
        lib.correct_kernel.argtypes = [P, P, P, I, F, I, P, P, P, P]
        lib.correct_kernel.restype = I
        lib.kv_rewrite.argtypes = [P, P, P]
        lib.kv_rewrite.restype = I
        lib.sirius_verify_row_argmax.argtypes = [P, P]
        lib.sirius_verify_row_argmax.restype = I
        lib.sirius_tree_kernel.argtypes = [P, P, P, I, I, I, F, I, P, P, P]
        lib.sirius_tree_kernel.restype = I
        lib.sirius_set_sampling.argtypes = [P, F, ctypes.c_uint64]
        lib.sirius_set_sampling.restype = I
        lib.sirius_topk_enable.argtypes = [P, F]
        lib.sirius_topk_enable.restype = I
        lib.sirius_par_export.argtypes = [P, P]
        lib.sirius_par_export.restype = I
        lib.sirius_par_enable.argtypes = [P, P]
        lib.sirius_par_enable.restype = I
        lib.sirius_par_disable.argtypes = [P]
        lib.sirius_par_disable.restype = I
        lib.sirius_csparse_enable.argtypes = [P, F]
        lib.sirius_csparse_enable.restype = I
        lib.sirius_debug_csparse_plan.argtypes = [P, P, P, ctypes.POINTER(I)]
        lib.sirius_debug_csparse_plan.restype = I
        lib.sirius_destroy.argtypes = [P]
        lib.sirius_destroy.restype = I
        lib.sirius_last_error.argtypes = [P]
        lib.sirius_last_error.restype = ctypes.c_char_p
        lib.sirius_version.argtypes = []
        lib.sirius_version.restype = ctypes.c_char_p
        lib.sirius_debug_gemm.argtypes = [P, I, I, P, P, P, I, I, I]
        lib.sirius_debug_ffn.argtypes = [P, I, P, I, P, P, P]
        lib.sirius_debug_ffn.restype = I
        lib.sirius_debug_buffer.argtypes = [P, I, I, P, ctypes.c_size_t]
        lib.sirius_debug_buffer.restype = I
        lib.sirius_debug_launches.argtypes = [P]
        lib.sirius_debug_launches.restype = ctypes.c_ulonglong
        lib.sirius_debug_trace_ffn.argtypes = [P, P, I]
        lib.sirius_debug_trace_ffn.restype = I
        lib.sirius_debug_trace_verify.argtypes = [P, P, I]
        lib.sirius_debug_trace_verify.restype = I
        lib.sirius_debug_trace.argtypes = [P, P]
        lib.sirius_debug_trace.restype = I
        lib.sirius_debug_graphs.argtypes = [P, I]
        lib.sirius_debug_graphs.restype = I
        lib.sirius_debug_profile.argtypes = [P, I]
        lib.sirius_debug_profile.restype = I
        lib.sirius_debug_profile_read.argtypes = [P, P, P]
        lib.sirius_debug_profile_read.restype = I
        lib.sirius_debug_gemm.restype = I
        lib.sirius_debug_par_skew.argtypes = [P, I, I]
        lib.sirius_debug_par_skew.restype = I
        lib.sirius_debug_topk.argtypes = [P, I, I, I, P, P]
        lib.sirius_debug_topk.restype = I
        lib.sirius_debug_gemv.argtypes = [P, I, I, P, I, P, P, P, P, P, P, P, I]
        lib.sirius_debug_gemv.restype = I
        lib.sirius_nccl_available.restype = I
        lib.sirius_nccl_unique_id.argtypes = [P]
        lib.sirius_nccl_unique_id.restype = I
        lib.sirius_nccl_comm_init.argtypes = [I, P, I, ctypes.POINTER(P)]
        lib.sirius_nccl_comm_init.restype = I
        lib.sirius_nccl_comm_destroy.argtypes = [P]
        lib.sirius_nccl_comm_destroy.restype = I
        _lib = lib
    return _lib


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Sirius:
    """One libsirius context (one GPU / TP rank, or a whole TP group emulated on one GPU)."""

    def __init__(self, cfg, weights, thresholds: Sequence[float], batch: int, max_seq: int, max_gamma: int,
                 tp_size: int = 1, tp_rank: int = 0, nccl_comm: Optional[int] = None, stream=None):
        import torch
        lib = load()
        if not torch.cuda.is_available():
            raise RuntimeError("libsirius needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.cfg = cfg
        self.batch, self.max_seq, self.max_gamma = batch, max_seq, max_gamma
        self.tp_size, self.tp_rank = tp_size, tp_rank
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        c = SiriusConfig(cfg.vocab, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim,
                         cfg.ffn_dim, cfg.rope_theta, cfg.rms_eps, batch, max_seq, max_gamma, tp_size, tp_rank)
        shards = weights if isinstance(weights, (list, tuple)) else [weights]
        self._keep = []  # keep ctypes arrays alive for the context's lifetime
        arr = (SiriusWeights * len(shards))()
        L = cfg.n_layers
        for i, w in enumerate(shards):
            per = {}
            for n in ("attn_norm", "w_qkv", "w_o", "ffn_norm", "w_gate", "w_up", "w_down"):
                a = (ctypes.c_void_p * L)(*[w[f"layers.{l}.{n}"].data_ptr() for l in range(L)])
                self._keep.append(a)
                per[n] = ctypes.cast(a, _PP)
            arr[i] = SiriusWeights(w["embed"].data_ptr(), w["final_norm"].data_ptr(), w["lm_head"].data_ptr(),
                                   per["attn_norm"], per["w_qkv"], per["w_o"], per["ffn_norm"], per["w_gate"],
                                   per["w_up"], per["w_down"])
        self._weights = shards
        thr = (ctypes.c_float * L)(*[float(t) for t in thresholds])
        h = ctypes.c_void_p()
        st = lib.sirius_init(ctypes.byref(c), arr, thr, nccl_comm, ctypes.c_void_p(self.stream.cuda_stream),
                             ctypes.byref(h))
        if st != SIRIUS_OK:
            raise SiriusError(st, "sirius_init failed")
        self.h = h
        self.lib = lib

    def _check(self, st: int):
        if st != SIRIUS_OK:
            raise SiriusError(st, self.lib.sirius_last_error(self.h).decode())

    def last_error(self) -> str:
        return self.lib.sirius_last_error(self.h).decode()

    # ---- C ABI, same names ------------------------------------------------------------
    def sirius_prefill(self, tokens, prompt_len: Sequence[int], first_token):
        lens = (ctypes.c_int32 * len(prompt_len))(*prompt_len)
        self._check(self.lib.sirius_prefill(self.h, _ptr(tokens), lens, _ptr(first_token)))

    def sparse_decode_step(self, token_in, pos, flags: int, token_out, logits_out=None, n_active_out=None,
                           gate_act_out=None):
        self._check(self.lib.sparse_decode_step(self.h, _ptr(token_in), _ptr(pos), flags, _ptr(token_out),
                                                _ptr(logits_out), _ptr(n_active_out), _ptr(gate_act_out)))

    def correct_kernel(self, kernel_tokens, start_pos, gamma: int, accept_threshold: float, accept_mode: int,
                       n_accept_out, next_token_out, q_out=None, logits_out=None):
        self._check(self.lib.correct_kernel(self.h, _ptr(kernel_tokens), _ptr(start_pos), gamma,
                                            accept_threshold, accept_mode, _ptr(n_accept_out),
                                            _ptr(next_token_out), _ptr(q_out), _ptr(logits_out)))

    def kv_rewrite(self, start_pos, n_rows):
        self._check(self.lib.kv_rewrite(self.h, _ptr(start_pos), _ptr(n_rows)))

    def sirius_verify_row_argmax(self, out):
        self._check(self.lib.sirius_verify_row_argmax(self.h, _ptr(out)))

    def sirius_tree_kernel(self, pending, start_pos, gamma: int, width: int, branch: int, accept_threshold: float,
                           accept_mode: int, n_accept_out, next_token_out, path_tokens_out):
        self._check(self.lib.sirius_tree_kernel(self.h, _ptr(pending), _ptr(start_pos), gamma, width, branch,
                                                accept_threshold, accept_mode, _ptr(n_accept_out),
                                                _ptr(next_token_out), _ptr(path_tokens_out)))

    def sirius_set_sampling(self, temperature: float, seed: int = 0):
        self._check(self.lib.sirius_set_sampling(self.h, float(temperature), int(seed) & (2 ** 64 - 1)))

    def sirius_topk_enable(self, keep_fraction: float):
        self._check(self.lib.sirius_topk_enable(self.h, float(keep_fraction)))

    def sirius_par_export(self) -> bytes:
        """This rank's comm-buffer IPC handle (SIRIUS_PAR_HANDLE_BYTES bytes) for sirius_par_enable."""
        buf = ctypes.create_string_buffer(PAR_HANDLE_BYTES)
        self._check(self.lib.sirius_par_export(self.h, buf))
        return buf.raw

    def sirius_par_enable(self, peer_handles: Optional[Sequence[bytes]] = None):
        """Fused NVLink peer all-reduce of the TP decode step.  peer_handles: every rank's exported
        handle in rank order (real ranks), None for emulated / stub contexts."""
        arg = None
        if peer_handles is not None:
            blob = b"".join(peer_handles)
            if len(blob) != PAR_HANDLE_BYTES * len(peer_handles):
                raise ValueError("each handle must be PAR_HANDLE_BYTES bytes")
            arg = ctypes.create_string_buffer(blob, len(blob))
        self._check(self.lib.sirius_par_enable(self.h, arg))

    def sirius_par_disable(self):
        self._check(self.lib.sirius_par_disable(self.h))

    def sirius_csparse_enable(self, keep_fraction: float):
        self._check(self.lib.sirius_csparse_enable(self.h, float(keep_fraction)))

    def debug_csparse_plan(self):
        """Test-only: (statistic fp32 [L, ffn/tp], plan int32 [L, k]) of the last prefill."""
        torch = self.torch
        k = ctypes.c_int32(0)
        self._check(self.lib.sirius_debug_csparse_plan(self.h, None, None, ctypes.byref(k)))
        L, F = self.cfg.n_layers, self.cfg.ffn_dim // self.tp_size
        stats = torch.zeros((L, F), dtype=torch.float32, device="cuda")
        idx = torch.zeros((L, k.value), dtype=torch.int32, device="cuda")
        self._check(self.lib.sirius_debug_csparse_plan(self.h, _ptr(stats), _ptr(idx), None))
        return stats, idx

    # ---- instrumentation (bench / tests) ------------------------------------------------
    def debug_ffn(self, layer: int, x, dense: bool, out, gate_out=None, n_active=None) -> None:
        """Test-only: the decode CATS FFN kernel of `layer` on residual rows x [batch, d] (fp32 CUDA)."""
        self._check(self.lib.sirius_debug_ffn(self.h, layer, _ptr(x), 1 if dense else 0, _ptr(out), _ptr(gate_out),
                                              _ptr(n_active)))

    PROF_NAMES = ("qkv_gemv", "attn_decode", "oproj_gemv", "cats_ffn", "lm_head", "correct_kernel", "kv_rewrite",
                  "decode_step")

    def launches(self) -> int:
        """Kernels this context has launched so far (library-side counter)."""
        return int(self.lib.sirius_debug_launches(self.h))

    def graphs(self, on: Optional[bool] = None) -> bool:
        """CUDA-graph replay of the ABI calls (default on); None = query."""
        return bool(self.lib.sirius_debug_graphs(self.h, -1 if on is None else (1 if on else 0)))

    def profile(self, on: bool) -> None:
        self.lib.sirius_debug_profile(self.h, 1 if on else 0)

    def profile_read(self) -> Dict[str, tuple]:
        """{kernel class: (total device ms, launches)} since profile(True); CUDA events on the
        library's stream around each launch."""
        tot = (ctypes.c_float * 8)()
        cnt = (ctypes.c_int * 8)()
        self.lib.sirius_debug_profile_read(self.h, tot, cnt)
        return {n: (float(tot[i]), int(cnt[i])) for i, n in enumerate(self.PROF_NAMES)}

    def sirius_destroy(self):
        if getattr(self, "h", None):
            self.lib.sirius_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.sirius_destroy()
        except Exception:
            pass


def debug_gemm(X, W, out, M: int, W2=None) -> None:
    """Test-only, via the tcgen05 kernel: X is bf16 [rows, K] (one term) or [nterms, rows, K] (term
    planes, x = their sum).  out = x[:M] @ W.T (fp32 [M, N]), or with W2 the SwiGLU
    m = SiLU(x W^T) * (x W2^T) as three bf16 term planes (out: bf16 [3, M, N])."""
    lib = load()
    N, K = W.shape
    nterms, rows = (1, X.shape[0]) if X.dim() == 2 else (X.shape[0], X.shape[1])
    r = lib.sirius_debug_gemm(X.data_ptr(), nterms, rows, W.data_ptr(), _ptr(W2), out.data_ptr(), M, N, K)
    if r != 0:
        raise RuntimeError(f"sirius_debug_gemm failed: {r}")


def debug_topk(g, k: int, a_out, mask) -> None:
    """Test-only: the top-k FSparse selection kernel on g (fp32 [B, F]): a_out [B, F] = SiLU(g), mask
    (int32 [B, F // 32 + 1], bit i of word i >> 5) = the k largest |a|, ties to the lower index."""
    lib = load()
    B, F = g.shape
    r = lib.sirius_debug_topk(g.data_ptr(), F, int(k), B, a_out.data_ptr(), mask.data_ptr())
    if r != 0:
        raise RuntimeError(f"sirius_debug_topk failed: {r}")


def debug_gemv(W, x, out, argmax=None, delta=None, norm_w=None, res_out=None, tokens=None, embed=None) -> None:
    """Test-only: out [B, rows] fp32 = h @ W.T (W bf16 [rows, K]) through the decode GEMV kernel;
    h = x (fp32 [B, K]); with norm_w (bf16 [K])
    h = RMSNorm(x + delta) * norm_w, res_out = x + delta; with embed (bf16 [V, K]) and tokens (int32 [B])
    h = RMSNorm(embed[tokens]) * norm_w (eps 1e-5); argmax: int32 [B] or None."""
    lib = load()
    rows, K = W.shape
    B = tokens.shape[0] if embed is not None else x.shape[0]
    r = lib.sirius_debug_gemv(W.data_ptr(), rows, K, _ptr(x), B, out.data_ptr(), _ptr(argmax), _ptr(delta), _ptr(norm_w), _ptr(res_out), _ptr(tokens), _ptr(embed),
                              embed.shape[0] if embed is not None else 0)
    if r != 0:
        raise RuntimeError(f"sirius_debug_gemv failed: {r}")
