"""Host driver of the Sirius loop (Algorithm 1) on top of the C ABI.

Host-side control flow and bookkeeping only: every arithmetic step (decode, verify, accept/reject,
KV rewrite) runs in libsirius kernels.  Per correction kernel there is one host<->device round trip:
the accepted count and the drafted tokens come back (D2H), the next kernel's positions and pending
tokens go out (H2D) — the "one host sync per kernel" of SURVEY.md CS1.

Modes (the three rows of the north-star metric):
  "dense"  : greedy decode with the full model M_F every token
  "sparse" : greedy decode with the CATS-sparse model M_S only (CS-only)
  "sirius" : M_S drafts gamma-1 tokens, M_F verifies the kernel, accept/reject, rewrite, interleave

Component ablation (Table 4; reading D27): Driver(..., rewrite, interleave,
rollback) switches KV Rewrite / Interleave / Rollback independently (rollback needs interleave).
Without rollback every kernel commits all gamma positions, a rejected draft replaced by the full
model's argmax of its verify row when interleaving (sirius_verify_row_argmax).
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
    advance: Optional[List[int]] = None  # per sequence, when not j + 1 (ablation without rollback)


@dataclass
class GenOut:
    tokens: List[List[int]]
    kernels: List[KernelLog] = field(default_factory=list)
    steps: int = 0  # decode steps launched

    def advances(self, b: int = 0) -> List[int]:
        return [int(k.j[b]) + 1 if k.advance is None else int(k.advance[b]) for k in self.kernels]

    def rejection_positions(self, b: int = 0) -> List[int]:
        """0-based draft index of every rejection (PAPER.md:678-685 histogram data)."""
        return [int(k.j[b]) for k in self.kernels if int(k.j[b]) < k.tokens.shape[1] - 1]


class Driver:
    def __init__(self, ctx: S.Sirius, rewrite: bool = True, interleave: bool = True, rollback: bool = True,
                 csparse: bool = False, topk: bool = False):
        """csparse: the draft model M_S is the CSparse model of the prompt (sirius_csparse_enable must
        have been called on ctx; the plan is built by every begin()) instead of CATS; topk: the top-k
        FSparse model (sirius_topk_enable)."""
        import torch
        assert interleave or not rollback, "rollback without interleave is not a Sirius configuration (Table 4)"
        self.rewrite, self.interleave, self.rollback = rewrite, interleave, rollback
        self.sparse_flags = S.SIRIUS_CSPARSE if csparse else (S.SIRIUS_TOPK if topk else 0)
        self.ctx, self.torch = ctx, torch
        B, gm = ctx.batch, ctx.max_gamma
        dev = "cuda"
        i32 = torch.int32
        self.B, self.gmax = B, gm
        self.drafts = torch.zeros((gm + 1, B), dtype=i32, device=dev)   # [i, b]: token_in of step i
        self.kbuf = torch.zeros((B, gm), dtype=i32, device=dev)         # kernel tokens [B, gamma]
        self.pos = torch.zeros((gm, B), dtype=i32, device=dev)          # positions of step i
        self.start = [torch.zeros(B, dtype=i32, device=dev) for _ in range(2)]  # ping-pong: this / previous kernel
        self.n_rows = torch.zeros(B, dtype=i32, device=dev)
        self.n_accept = torch.zeros(B, dtype=i32, device=dev)
        self.next_tok = torch.zeros(B, dtype=i32, device=dev)
        self.q = torch.zeros((B, gm), dtype=torch.float32, device=dev)
        self.row_am = torch.zeros((B, gm), dtype=torch.int32, device=dev)
        self.path = torch.zeros(gm, dtype=torch.int32, device=dev)  # tree kernels: winning path tokens
        # pinned staging: out = [n_rows(B) | start(B) | pending(B) | pos(gm*B)], in = [n_accept | next | drafts]
        self.h_out = torch.zeros(3 * B + gm * B, dtype=i32).pin_memory()
        self.h_in = torch.zeros(2 * B + (gm + 1) * B, dtype=i32).pin_memory()
        self.d_out = torch.zeros(3 * B + gm * B, dtype=i32, device=dev)
        self.d_in = torch.zeros(2 * B + (gm + 1) * B, dtype=i32, device=dev)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self._h_out_ev = None  # recorded after the last H2D copy out of h_out

    # ------------------------------------------------------------------ session state
    def begin(self, prompts: Sequence[Sequence[int]]) -> None:
        """Dense prefill; the first generated token is the dense argmax (reading D17)."""
        torch = self.torch
        flat = torch.tensor(np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts]), device="cuda")
        first = torch.zeros(self.B, dtype=torch.int32, device="cuda")
        self.ctx.sirius_prefill(flat, [len(p) for p in prompts], first)
        first = first.cpu().tolist()
        self.T = [len(p) for p in prompts]
        self.out = [[f] for f in first]
        self.pending = list(first)
        self.n_rows_h = [0] * self.B
        self.need_rewrite = False
        self.kidx = 0
        self.log: List[KernelLog] = []

    def _upload(self, gamma: int, T=None) -> None:
        B = self.B
        T = self.T if T is None else T
        # the previous non-blocking copy out of the pinned h_out may still be queued behind earlier
        # steps: wait for it before overwriting h_out (it runs ahead of the steps enqueued after it,
        # so the stream keeps those queued meanwhile)
        if self._h_out_ev is not None:
            self._h_out_ev.synchronize()
        h = self.h_out.numpy()
        h[0:B] = self.n_rows_h
        h[B:2 * B] = T
        h[2 * B:3 * B] = self.pending
        pos = (np.asarray(T, dtype=np.int64)[None, :] + np.arange(gamma)[:, None]).astype(np.int32)
        h[3 * B:3 * B + gamma * B] = pos.reshape(-1)
        n = 3 * B + gamma * B
        self.d_out[:n].copy_(self.h_out[:n], non_blocking=True)
        self._h_out_ev = self.torch.cuda.Event()
        self._h_out_ev.record()
        self.h2d_bytes += 4 * n

    def flush(self) -> None:
        """Commit the last kernel's rows (kv_rewrite) and wait for the stream."""
        if self.need_rewrite:
            B = self.B
            self._upload(1)
            self.n_rows.copy_(self.d_out[0:B])
            self.ctx.kv_rewrite(self.start[(self.kidx - 1) % 2], self.n_rows)
            self.need_rewrite = False
        self.torch.cuda.current_stream().synchronize()

    def step(self, gamma: int, r: float, accept_mode: int = S.ACCEPT_THRESHOLD, keep_q: bool = False) -> int:
        """One correction kernel (kernel size gamma): M_S drafts gamma-1 tokens, M_F verifies,
        accept/reject + interleave; the previous kernel's KV rewrite is enqueued first.  Returns the
        number of tokens committed for sequence 0."""
        torch, B = self.torch, self.B
        assert 1 <= gamma <= self.gmax
        self._upload(gamma)
        d = self.d_out
        cur = self.start[self.kidx % 2]
        self.n_rows.copy_(d[0:B])
        cur.copy_(d[B:2 * B])
        self.drafts[0].copy_(d[2 * B:3 * B])
        self.pos[:gamma].copy_(d[3 * B:3 * B + gamma * B].view(gamma, B))
        if self.need_rewrite:  # commit + rollback of the previous kernel
            self.ctx.kv_rewrite(self.start[(self.kidx - 1) % 2], self.n_rows)
        for i in range(gamma - 1):  # M_S drafts gamma-1 tokens (Alg. 1 lines 6-11)
            self.ctx.sparse_decode_step(self.drafts[i], self.pos[i], self.sparse_flags, self.drafts[i + 1])
        if B == 1:
            kt = self.drafts[:gamma].view(1, gamma)
        else:
            self.kbuf[:, :gamma].copy_(self.drafts[:gamma].t())
            kt = self.kbuf[:, :gamma].contiguous()
        ablate = not self.rollback
        self.ctx.correct_kernel(kt, cur, gamma, r, accept_mode, self.n_accept, self.next_tok,
                                self.q if (keep_q or ablate) else None)
        if ablate:
            self.ctx.sirius_verify_row_argmax(self.row_am)
        # D2H: accepted count, interleaved token, drafts (the one sync per kernel)
        n = 2 * B + gamma * B
        self.d_in[0:B].copy_(self.n_accept)
        self.d_in[B:2 * B].copy_(self.next_tok)
        self.d_in[2 * B:n].copy_(self.drafts[:gamma].reshape(-1))
        self.h_in[:n].copy_(self.d_in[:n], non_blocking=True)
        self.d2h_bytes += 4 * n
        torch.cuda.current_stream().synchronize()
        h = self.h_in.numpy()
        j = h[0:B].copy()
        nxt = h[B:2 * B].copy()
        dr = h[2 * B:n].reshape(gamma, B)
        qh = self.q[:, :gamma].cpu().numpy() if (keep_q or ablate) else None
        self.log.append(KernelLog(list(self.T), dr.T.copy(), j, nxt, qh))
        am = self.row_am[:, :gamma].cpu().numpy() if ablate else None
        advs = []
        for b in range(B):
            jb = int(j[b])
            if self.rollback:  # commit + rollback to the first rejection; interleave the full model's token
                committed = [int(x) for x in dr[1:jb + 1, b]] + [int(nxt[b])]
            else:  # no rollback: all gamma positions; rejected drafts interleaved (or kept)
                committed = []
                for i in range(gamma - 1):
                    d_i = int(dr[i + 1, b])
                    ok = (qh[b, i] >= r) if accept_mode == S.ACCEPT_THRESHOLD else (d_i == int(am[b, i]))
                    committed.append(d_i if (ok or not self.interleave) else int(am[b, i]))
                committed.append(int(am[b, gamma - 1]))
            self.out[b] += committed
            advs.append(len(committed))
            self.n_rows_h[b] = len(committed)
            self.T[b] += len(committed)
            self.pending[b] = committed[-1]
        self.log[-1].advance = None if self.rollback else advs
        self.need_rewrite = self.rewrite
        self.kidx += 1
        return advs[0]

    def step_tree(self, gamma: int, r: float, width: int, branch: int = 3,
                  accept_mode: int = S.ACCEPT_THRESHOLD) -> int:
        """One tree correction kernel (sirius_tree_kernel: tree drafting + tree verification, PAPER.md:
        299-319); batch 1.  Same host round trip as step(): the accepted count, the interleaved token and
        the winning path's tokens come back; the commit (kv_rewrite of the path) is enqueued next time."""
        torch = self.torch
        assert self.B == 1 and self.rollback and self.interleave
        self._upload(gamma)
        d = self.d_out
        cur = self.start[self.kidx % 2]
        self.n_rows.copy_(d[0:1])
        cur.copy_(d[1:2])
        self.drafts[0].copy_(d[2:3])
        if self.need_rewrite:
            self.ctx.kv_rewrite(self.start[(self.kidx - 1) % 2], self.n_rows)
        self.ctx.sirius_tree_kernel(self.drafts[0], cur, gamma, width, branch, r, accept_mode, self.n_accept,
                                    self.next_tok, self.path)
        n = 2 + gamma
        self.d_in[0:1].copy_(self.n_accept)
        self.d_in[1:2].copy_(self.next_tok)
        self.d_in[2:n].copy_(self.path[:gamma])
        self.h_in[:n].copy_(self.d_in[:n], non_blocking=True)
        self.d2h_bytes += 4 * n
        torch.cuda.current_stream().synchronize()
        h = self.h_in.numpy()
        j, nxt = int(h[0]), int(h[1])
        path = h[2:n].copy()
        self.log.append(KernelLog(list(self.T), path[None, :].copy(), np.array([j]), np.array([nxt])))
        committed = [int(x) for x in path[1:j + 1]] + [nxt]
        self.out[0] += committed
        self.n_rows_h[0] = len(committed)
        self.T[0] += len(committed)
        self.pending[0] = committed[-1]
        self.need_rewrite = True
        self.kidx += 1
        return len(committed)

    def sirius_tree(self, prompts, n_tokens: int, gamma: int, r: float, width: int, branch: int = 3,
                    accept_mode: int = S.ACCEPT_THRESHOLD) -> GenOut:
        self.begin(prompts)
        while len(self.out[0]) < n_tokens:
            self.step_tree(gamma, r, width, branch, accept_mode)
        self.flush()
        return GenOut([o[:n_tokens] for o in self.out], list(self.log))

    # ------------------------------------------------------------------ whole generations
    def sirius(self, prompts, n_tokens: int, gamma: int, r: float, accept_mode: int = S.ACCEPT_THRESHOLD,
               keep_q: bool = False) -> GenOut:
        self.begin(prompts)
        while min(len(o) for o in self.out) < n_tokens:
            self.step(gamma, r, accept_mode, keep_q)
        self.flush()
        return GenOut([o[:n_tokens] for o in self.out], list(self.log))

    def greedy(self, prompts, n_tokens: int, dense: bool) -> GenOut:
        """Plain greedy decode (dense M_F or CS-only M_S) after a dense prefill."""
        torch, B = self.torch, self.B
        self.begin(prompts)
        P = self.T
        toks = torch.zeros((n_tokens, B), dtype=torch.int32, device="cuda")
        toks[0] = torch.tensor(self.pending, dtype=torch.int32)
        pos = torch.tensor(np.array([[P[b] + i for b in range(B)] for i in range(n_tokens)], dtype=np.int32),
                           device="cuda")
        self.greedy_steps(toks, pos, n_tokens - 1, dense)
        host = toks.cpu().numpy()
        return GenOut([host[:, b].tolist() for b in range(B)], steps=n_tokens - 1)

    def greedy_steps(self, toks, pos, n: int, dense: bool, first: int = 0) -> None:
        flags = S.SIRIUS_DENSE if dense else self.sparse_flags
        for i in range(first, first + n):
            self.ctx.sparse_decode_step(toks[i], pos[i], flags, toks[i + 1])

    def greedy_run(self, pending, T, n: int, dense: bool) -> None:
        """n greedy decode steps (dense M_F or CS-only M_S) continuing from `pending` at positions
        T, T+1, ...: chunks of max_gamma steps over fixed buffer slots (so each step replays a cached
        CUDA graph), one H2D of the chunk's positions per chunk, no host sync."""
        B, m = self.B, self.gmax
        flags = S.SIRIUS_DENSE if dense else self.sparse_flags
        T = list(T)
        self.drafts[0].copy_(self.torch.tensor(pending, dtype=self.torch.int32), non_blocking=False)
        done = 0
        while done < n:
            k = min(m, n - done)
            self._upload(m, T)  # positions T .. T + m - 1 of this chunk into d_out
            self.pos[:m].copy_(self.d_out[3 * B:3 * B + m * B].view(m, B))
            for i in range(k):
                self.ctx.sparse_decode_step(self.drafts[i], self.pos[i], flags, self.drafts[i + 1])
            self.drafts[0].copy_(self.drafts[k])
            T = [t + k for t in T]
            done += k
