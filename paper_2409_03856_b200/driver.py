"""Host driver of the Sirius loop (Algorithm 1) on top of the C ABI.

Host-side control flow and bookkeeping only: every arithmetic step (decode, verify, accept/reject,
KV rewrite) runs in libsirius kernels.  Per correction kernel there is one host<->device round trip:
the accepted count and the drafted tokens come back (D2H), the next kernel's positions and pending
tokens go out (H2D) — the "one host sync per kernel" of SURVEY.md CS1.

Modes (the three rows of the north-star metric):
  "dense"  : greedy decode with the full model M_F every token
  "sparse" : greedy decode with the CATS-sparse model M_S only (CS-only)
  "sirius" : M_S drafts gamma-1 tokens, M_F verifies the kernel, accept/reject, rewrite, interleave
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import sirius as S


@dataclass
class KernelLog:
    T: List[int]
    tokens: np.ndarray  # [B, gamma]
    j: np.ndarray       # [B]
    next_token: np.ndarray
    q: Optional[np.ndarray] = None


@dataclass
class GenOut:
    tokens: List[List[int]]
    kernels: List[KernelLog] = field(default_factory=list)
    steps: int = 0  # decode steps launched

    def advances(self, b: int = 0) -> List[int]:
        return [int(k.j[b]) + 1 for k in self.kernels]


class Driver:
    def __init__(self, ctx: S.Sirius):
        import torch
        self.ctx, self.torch = ctx, torch
        B, gm = ctx.batch, ctx.max_gamma
        dev = "cuda"
        i32 = torch.int32
        self.B, self.gmax = B, gm
        self.drafts = torch.zeros((gm + 1, B), dtype=i32, device=dev)   # [i, b]: token_in of step i
        self.kbuf = torch.zeros((B, gm), dtype=i32, device=dev)         # kernel tokens [B, gamma]
        self.pos = torch.zeros((gm, B), dtype=i32, device=dev)          # positions of step i
        self.start = torch.zeros(B, dtype=i32, device=dev)
        self.n_rows = torch.zeros(B, dtype=i32, device=dev)
        self.n_accept = torch.zeros(B, dtype=i32, device=dev)
        self.next_tok = torch.zeros(B, dtype=i32, device=dev)
        self.q = torch.zeros((B, gm), dtype=torch.float32, device=dev)
        # pinned staging: [n_rows(B) | start(B) | drafts0(B) | pos(gm*B)] out, [n_accept | next | drafts] in
        self.h_out = torch.zeros(3 * B + gm * B, dtype=i32).pin_memory()
        self.h_in = torch.zeros(2 * B + (gm + 1) * B, dtype=i32).pin_memory()
        self.d_out = torch.zeros(3 * B + gm * B, dtype=i32, device=dev)
        self.d_in = torch.zeros(2 * B + (gm + 1) * B, dtype=i32, device=dev)

    # ------------------------------------------------------------------ helpers
    def prefill(self, prompts: Sequence[Sequence[int]]) -> List[int]:
        torch = self.torch
        flat = torch.tensor(np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts]), device="cuda")
        first = torch.zeros(self.B, dtype=torch.int32, device="cuda")
        self.ctx.sirius_prefill(flat, [len(p) for p in prompts], first)
        return first.cpu().tolist()

    def _upload(self, n_rows, start, pending, T, gamma):
        B = self.B
        h = self.h_out.numpy()
        h[0:B] = n_rows
        h[B:2 * B] = start
        h[2 * B:3 * B] = pending
        pos = (np.asarray(T, dtype=np.int64)[None, :] + np.arange(gamma)[:, None]).astype(np.int32)
        h[3 * B:3 * B + gamma * B] = pos.reshape(-1)
        self.d_out[:3 * B + gamma * B].copy_(self.h_out[:3 * B + gamma * B], non_blocking=True)

    # ------------------------------------------------------------------ baselines
    def greedy(self, prompts, n_tokens: int, dense: bool) -> GenOut:
        """Plain greedy decode (dense M_F or CS-only M_S) after a dense prefill."""
        torch, B = self.torch, self.B
        first = self.prefill(prompts)
        P = [len(p) for p in prompts]
        out = [[f] for f in first]
        toks = torch.zeros((n_tokens, B), dtype=torch.int32, device="cuda")
        toks[0] = torch.tensor(first, dtype=torch.int32)
        pos = torch.tensor(np.array([[P[b] + i for b in range(B)] for i in range(n_tokens)], dtype=np.int32),
                           device="cuda")
        flags = S.SIRIUS_DENSE if dense else 0
        for i in range(n_tokens - 1):
            self.ctx.sparse_decode_step(toks[i], pos[i], flags, toks[i + 1])
        host = toks.cpu().numpy()
        for b in range(B):
            out[b] = host[:, b].tolist()
        return GenOut(out, steps=n_tokens - 1)

    # ------------------------------------------------------------------ Sirius
    def sirius(self, prompts, n_tokens: int, gamma: int, r: float, accept_mode: int = S.ACCEPT_THRESHOLD,
               keep_q: bool = False) -> GenOut:
        torch, B = self.torch, self.B
        assert 1 <= gamma <= self.gmax
        first = self.prefill(prompts)
        T = [len(p) for p in prompts]
        out = [[f] for f in first]
        res = GenOut(out)
        pending = list(first)
        n_rows = [0] * B
        first_kernel = True
        while min(len(o) for o in out) < n_tokens:
            # H2D: previous kernel's n_rows, this kernel's start / pending token / positions
            self._upload(n_rows, T, pending, T, gamma)
            d = self.d_out
            self.n_rows.copy_(d[0:B])
            self.start.copy_(d[B:2 * B])
            self.drafts[0].copy_(d[2 * B:3 * B])
            self.pos[:gamma].copy_(d[3 * B:3 * B + gamma * B].view(gamma, B))
            if not first_kernel:  # commit + rollback of the previous kernel
                self.ctx.kv_rewrite(self.prev_start, self.n_rows)
            for i in range(gamma - 1):  # M_S drafts gamma-1 tokens (Alg. 1 lines 6-11)
                self.ctx.sparse_decode_step(self.drafts[i], self.pos[i], 0, self.drafts[i + 1])
                res.steps += 1
            if B == 1:
                kt = self.drafts[:gamma].view(1, gamma)
            else:
                self.kbuf[:, :gamma].copy_(self.drafts[:gamma].t())
                kt = self.kbuf[:, :gamma].contiguous()
            self.ctx.correct_kernel(kt, self.start, gamma, r, accept_mode, self.n_accept, self.next_tok,
                                    self.q if keep_q else None)
            # D2H: accepted count, interleaved token, drafts (one sync per kernel)
            self.d_in[0:B].copy_(self.n_accept)
            self.d_in[B:2 * B].copy_(self.next_tok)
            self.d_in[2 * B:2 * B + gamma * B].copy_(self.drafts[:gamma].reshape(-1))
            self.h_in[:2 * B + gamma * B].copy_(self.d_in[:2 * B + gamma * B], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            h = self.h_in.numpy()
            j = h[0:B].copy()
            nxt = h[B:2 * B].copy()
            dr = h[2 * B:2 * B + gamma * B].reshape(gamma, B)
            kl = KernelLog(list(T), dr.T.copy(), j, nxt, self.q[:, :gamma].cpu().numpy() if keep_q else None)
            res.kernels.append(kl)
            self.prev_start = self.start.clone()
            for b in range(B):
                jb = int(j[b])
                out[b] += [int(x) for x in dr[1:jb + 1, b]] + [int(nxt[b])]
                n_rows[b] = jb + 1
                T[b] += jb + 1
                pending[b] = int(nxt[b])
            first_kernel = False
        # final commit of the last kernel
        self._upload(n_rows, T, pending, T, 1)
        self.n_rows.copy_(self.d_out[0:B])
        self.ctx.kv_rewrite(self.prev_start, self.n_rows)
        torch.cuda.current_stream().synchronize()
        res.tokens = [o[:n_tokens] for o in out]
        return res
