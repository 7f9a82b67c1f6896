"""CPU ORACLE for the Sirius decode hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It shares no code with the CUDA
path (``paper_2409_03856_b200``) and never takes an input or expected value from it.

Layers:
  * ``oracle.cpp`` (fp64, plain loops): one decoder row (``forward_row``), the layer MLP
    with CATS thresholding, KV rewrite.  See its header for the citations and the
    numeric contract (D15).
  * this file: the Sirius loop, Algorithm 1 with the readings
    D5-D14, D17-D18 of DESIGN.md §2, written out step by step; plus the paper's
    efficiency formulas (Eq. 1-3) and the SD expected-AAL formula
    (PAPER.md:100-104).

Pins (tests/test_oracle_*.py): HF LlamaForCausalLM fp64; KV identity; chunk == sequential;
brute-force masked MLP; t=0 == dense; r=0 accepts all; EXACT_ARGMAX == dense greedy;
rewrite equivalence; accounting identities; Table 2 / §5.2 / §2.3 printed arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ACCEPT_THRESHOLD = 0  # keep d_{i+1} iff q_i = softmax(l_i)[d_{i+1}] >= r  (reading D14)
ACCEPT_EXACT_ARGMAX = 1  # keep d_{i+1} iff d_{i+1} == argmax l_i (speculative-decoding greedy match)


def build() -> str:
    out = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.cpp")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                               "-o", out, src])
    return out


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.oracle_create.argtypes = [ctypes.c_int] * 7 + [ctypes.c_double, ctypes.c_double] + [ctypes.c_int] * 4
        lib.oracle_create.restype = P
        lib.oracle_destroy.argtypes = [P]
        lib.oracle_set_global.argtypes = [P, P, P, P]
        lib.oracle_set_layer.argtypes = [P, ctypes.c_int] + [P] * 7
        lib.oracle_forward_row.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, P, P, P, P,
                                           P, ctypes.c_uint64, ctypes.c_int]
        lib.oracle_kv_rewrite_rows.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_prefill_kv_row.argtypes = [P, ctypes.c_int, ctypes.c_int]
        lib.oracle_mlp.argtypes = [P, ctypes.c_int, P, ctypes.c_int, ctypes.c_float, P, P, P, P]
        lib.oracle_kv_rewrite.argtypes = [P, ctypes.c_int, ctypes.c_int]
        lib.oracle_read_cache.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P]
        lib.oracle_round_bf16.argtypes = [ctypes.c_double]
        lib.oracle_round_bf16.restype = ctypes.c_double
        _LIB = lib
    return _LIB


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def round_bf16(x: float) -> float:
    return float(_lib().oracle_round_bf16(float(x)))


@dataclass
class RowOut:
    logits: np.ndarray  # fp64 [vocab]
    gate: Optional[np.ndarray] = None  # a = SiLU(g), fp64 [L, ffn]
    mask: Optional[np.ndarray] = None  # uint8 [L, ffn]
    n_active: Optional[np.ndarray] = None  # int32 [L]


class OracleModel:
    """One sequence's oracle state: borrowed weights + its own KV cache and staging."""

    def __init__(self, cfg, weights: Dict[str, np.ndarray], max_seq: int, max_gamma: int = 64,
                 threads: Optional[int] = None, round_kv: bool = True):
        self.cfg = cfg
        self.w = weights  # keep alive
        self.max_seq, self.max_gamma = max_seq, max_gamma
        self.threads = threads or max(1, os.cpu_count() or 1)
        lib = _lib()
        self.h = lib.oracle_create(cfg.vocab, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim,
                                   cfg.ffn_dim, cfg.rope_theta, cfg.rms_eps, max_seq, max_gamma, self.threads,
                                   1 if round_kv else 0)
        for k in weights:
            assert weights[k].dtype == np.uint16 and weights[k].flags["C_CONTIGUOUS"], k
        lib.oracle_set_global(self.h, _ptr(weights["embed"]), _ptr(weights["final_norm"]), _ptr(weights["lm_head"]))
        for l in range(cfg.n_layers):
            g = lambda n: _ptr(weights[f"layers.{l}.{n}"])
            lib.oracle_set_layer(self.h, l, g("attn_norm"), g("w_qkv"), g("w_o"), g("ffn_norm"), g("w_gate"),
                                 g("w_up"), g("w_down"))

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h and _LIB is not None:
            try:
                _LIB.oracle_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    # ------------------------------------------------------------ one row
    def forward_row(self, tok: int, pos: int, sparse: bool = False, thresholds: Optional[np.ndarray] = None,
                    stage_row: int = -1, want_gate: bool = False, want_mask: bool = False,
                    plan: Optional[np.ndarray] = None, tree_vis: int = 0, tree_n_cache: int = 0,
                    topk: Optional[np.ndarray] = None) -> RowOut:
        """sparse with plan (uint8 [L, ffn], csparse_plan): the CSparse model; sparse with topk (keep
        fraction per layer): the top-k FSparse model (reading D30); sparse with thresholds: the CATS
        (FSparse) model; else the dense model."""
        cfg = self.cfg
        assert 0 <= tok < cfg.vocab and 0 <= pos < self.max_seq
        assert stage_row < self.max_gamma
        logits = np.empty(cfg.vocab, dtype=np.float64)
        gate = np.empty((cfg.n_layers, cfg.ffn_dim), dtype=np.float64) if want_gate else None
        mask = np.empty((cfg.n_layers, cfg.ffn_dim), dtype=np.uint8) if want_mask else None
        nact = np.empty(cfg.n_layers, dtype=np.int32)
        thr = pl = None
        mode = 0
        if sparse and topk is not None:
            thr = np.ascontiguousarray(topk, dtype=np.float32)
            assert thr.shape == (cfg.n_layers,)
            mode = 3
        elif sparse and plan is not None:
            pl = np.ascontiguousarray(plan, dtype=np.uint8)
            assert pl.shape == (cfg.n_layers, cfg.ffn_dim)
            mode = 2
        elif sparse:
            thr = np.ascontiguousarray(thresholds, dtype=np.float32)
            assert thr.shape == (cfg.n_layers,)
            mode = 1
        _lib().oracle_forward_row(self.h, int(tok), int(pos), mode, _ptr(thr), int(stage_row),
                                  _ptr(logits), _ptr(gate), _ptr(mask), _ptr(nact), None, _ptr(pl),
                                  int(tree_vis), int(tree_n_cache))
        return RowOut(logits, gate, mask, nact)

    def mlp(self, layer: int, x: np.ndarray, sparse: bool, threshold: float = 0.0, plan: Optional[np.ndarray] = None,
            topk: Optional[float] = None):
        """Layer-isolated MLP on residual x (fp64 [d]); returns (x_out, a, mask, n_active).  With plan
        (uint8 [ffn]) the CSparse MLP of that neuron set."""
        cfg = self.cfg
        xx = np.ascontiguousarray(x, dtype=np.float64).copy()
        gate = np.empty(cfg.ffn_dim, dtype=np.float64)
        mask = np.empty(cfg.ffn_dim, dtype=np.uint8)
        n = np.empty(1, dtype=np.int32)
        pl = None if plan is None else np.ascontiguousarray(plan, dtype=np.uint8)
        mode = 3 if (sparse and topk is not None) else (2 if (sparse and pl is not None) else (1 if sparse else 0))
        _lib().oracle_mlp(self.h, layer, _ptr(xx), mode, float(topk if mode == 3 else threshold), _ptr(gate),
                          _ptr(mask), _ptr(n), _ptr(pl))
        return xx, gate, mask, int(n[0])

    def kv_rewrite(self, T: int, n: int) -> None:
        assert 1 <= n <= self.max_gamma and T + n <= self.max_seq
        _lib().oracle_kv_rewrite(self.h, int(T), int(n))

    def kv_rewrite_rows(self, T: int, rows: Sequence[int]) -> None:
        """Commit staging rows `rows` (in order) into cache slots [T, T + len(rows)) (tree commit)."""
        r = np.ascontiguousarray(rows, dtype=np.int32)
        assert 1 <= len(r) and T + len(r) <= self.max_seq and r.max() < self.max_gamma
        _lib().oracle_kv_rewrite_rows(self.h, int(T), len(r), _ptr(r))

    def read_cache(self, layer: int, n: int):
        cfg = self.cfg
        k = np.empty((n, cfg.n_kv_heads, cfg.head_dim), dtype=np.float64)
        v = np.empty_like(k)
        _lib().oracle_read_cache(self.h, layer, n, _ptr(k), _ptr(v))
        return k, v

    # ------------------------------------------------------------ model-level steps
    def prefill(self, tokens: Sequence[int]) -> np.ndarray:
        """Dense prefill (PAPER.md:471 'most use full weights for prefilling', reading D17).
        Writes the cache rows [0, P); returns the logits of every prompt position [P, vocab]."""
        return np.stack([self.forward_row(t, i).logits for i, t in enumerate(tokens)])

    def prefill_last(self, tokens: Sequence[int]) -> np.ndarray:
        """Dense prefill that returns only the last position's logits: rows [0, P-1) write their
        K/V cache rows only (oracle_prefill_kv_row), the last row runs in full.  Same cache
        contents as prefill(); used where long prompts would make the full version slow."""
        lib = _lib()
        for i, t in enumerate(tokens[:-1]):
            assert 0 <= t < self.cfg.vocab and i < self.max_seq
            lib.oracle_prefill_kv_row(self.h, int(t), i)
        return self.forward_row(tokens[-1], len(tokens) - 1).logits

    def prefill_stats(self, tokens: Sequence[int]):
        """Dense prefill that also returns the CSparse statistic of every layer's neurons over the
        prompt (§2.1 "the sparsity pattern is fixed for all tokens generated", decided
        after prefilling; reading D28): stats[l, i] = sum over prompt positions p of
        |a_{p,i}|, a = SiLU(g) of the dense model.  Returns (logits [P, vocab], stats [L, ffn])."""
        stats = np.zeros((self.cfg.n_layers, self.cfg.ffn_dim), dtype=np.float64)
        logits = []
        for i, t in enumerate(tokens):
            row = self.forward_row(t, i, want_gate=True)
            stats += np.abs(row.gate)
            logits.append(row.logits)
        return np.stack(logits), stats

    def decode(self, tok: int, pos: int, sparse: bool, thresholds=None, **kw) -> RowOut:
        """One decode step of M_S (sparse) or M_F (dense): writes K/V at cache slot pos."""
        return self.forward_row(tok, pos, sparse, thresholds, -1, **kw)

    def verify(self, kernel_tokens: Sequence[int], T: int) -> np.ndarray:
        """Full-model parallel verification of one kernel (Alg. 1 line 'FORWARD(M_F, C, kernel)',
        PAPER.md:258; §4.2): rows [pending, d_1..d_{g-1}] at positions T..T+g-1,
        K/V into staging, each row attends to cache[0,T) + staging[0..i].  Returns logits [g, vocab]."""
        return np.stack([self.forward_row(t, T + i, False, None, i).logits for i, t in enumerate(kernel_tokens)])


def csparse_keep_count(ffn: int, keep: float) -> int:
    """Neurons kept per layer: round(keep * ffn), halves rounded up (reading D28)."""
    return int(np.floor(keep * ffn + 0.5))


def csparse_plan(stats: np.ndarray, keep: float) -> np.ndarray:
    """CSparse neuron plan (reading D28): per layer the csparse_keep_count(ffn, keep) neurons with
    the largest statistic, exact ties to the lower neuron index.  Returns uint8 [L, ffn] (1 = kept)."""
    L, F = stats.shape
    k = csparse_keep_count(F, keep)
    plan = np.zeros((L, F), dtype=np.uint8)
    idx = np.arange(F)
    for l in range(L):
        order = np.lexsort((idx, -stats[l]))  # primary: statistic descending; secondary: index ascending
        plan[l, order[:k]] = 1
    return plan


_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 output function of state x (Steele, Lea, Flood 2014): the counter-based generator of
    the sampled tokens (reading D31)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def sample_uniform(seed: int, b: int, p: int) -> float:
    """u for the token placed at absolute position p of sequence b: 24 bits, exact in fp32."""
    return float(splitmix64((seed ^ splitmix64(((b << 32) + p) & _M64)) & _M64) >> 40) / 16777216.0


def sample_token(l: np.ndarray, temperature: float, u: float) -> int:
    """Inverse CDF of softmax(l / temperature) in index order (PAPER.md:253, :267 'sample'; reading
    D31): the smallest v with sum_{w <= v} e_w > u Z, e_w = exp((l_w - max l) / T)."""
    e = np.exp((l - l.max()) / temperature)
    c = np.cumsum(e)
    v = int(np.searchsorted(c, u * c[-1], side="right"))
    if v >= l.size:
        v = int(np.flatnonzero(e > 0)[-1])
    return v


def sample_margin(l: np.ndarray, temperature: float, u: float) -> float:
    """Relative distance of u Z to the nearest CDF boundary (ambiguity of a sampled token under float
    error, the sampling analogue of the top-2 margin)."""
    e = np.exp((l - l.max()) / temperature)
    c = np.cumsum(e)
    t = u * c[-1]
    return float(np.min(np.abs(c - t)) / c[-1])


def top2_margin(l: np.ndarray) -> float:
    """Largest minus second-largest logit (0 on an exact tie): how far the argmax is from flipping."""
    s = np.partition(l, -2)[-2:]
    return float(s[1] - s[0])


def argmax_lowest(l: np.ndarray) -> int:
    """argmax with the lowest token id on exact ties (reading D13)."""
    return int(np.flatnonzero(l == l.max())[0])


def softmax_prob(l: np.ndarray, tok: int) -> float:
    """q = softmax(l)[tok] at temperature 1 (reading D12)."""
    m = l.max()
    return float(np.exp(l[tok] - m) / np.exp(l - m).sum())


def accept_scan(lf: np.ndarray, kernel_tokens: Sequence[int], r: float, mode: int = ACCEPT_THRESHOLD):
    """Algorithm 1 lines 'for j from 0, n: if q_{t+j} < r: break', reading D8/D14.
    Returns (j, q): j = first rejected index in [0, g-2], or g-1 if all g-1 drafts are accepted;
    q[i] = full-model probability of draft d_{i+1} for i < g-1, q[g-1] = probability of argmax row g-1."""
    g = len(kernel_tokens)
    q = np.empty(g, dtype=np.float64)
    j = g - 1
    for i in range(g - 1):
        q[i] = softmax_prob(lf[i], kernel_tokens[i + 1])
    q[g - 1] = softmax_prob(lf[g - 1], argmax_lowest(lf[g - 1]))
    for i in range(g - 1):
        ok = q[i] >= r if mode == ACCEPT_THRESHOLD else kernel_tokens[i + 1] == argmax_lowest(lf[i])
        if not ok:
            j = i
            break
    return j, q


@dataclass
class KernelRecord:
    T: int  # cache length before the kernel (position of the pending token)
    tokens: List[int]  # [pending, d_1..d_{g-1}]
    j: int  # accepted drafts (= first rejected index, or g-1)
    q: np.ndarray  # full-model likelihoods
    next_token: int  # interleaved / bonus token = argmax of verify row j
    n_active: np.ndarray  # [g-1, L] active neurons per sparse step
    draft_margin: np.ndarray = None   # [g-1] top-2 logit margin of each sparse drafting row
    verify_margin: np.ndarray = None  # [g] top-2 logit margin of each verify row
    advance: int = 0                  # tokens committed by this kernel (j + 1 with rollback, else g)
    tree: Optional["TreeKernel"] = None  # the tree of a tree kernel (tree_width given)


def log_softmax(l: np.ndarray) -> np.ndarray:
    m = l.max()
    return l - (m + np.log(np.exp(l - m).sum()))


@dataclass
class TreeKernel:
    """One tree correction kernel (reading D29).  Flattened rows:
    0 = the pending token at position T; node w of step s (1 <= s <= gamma-1) = row 1 + (s-1) W + w at
    position T + s."""
    tokens: List[int]
    parent: List[int]
    cum: List[float]        # cumulative sparse log-likelihood of the node's path (root 0)
    vis: List[int]          # 64-bit ancestor-or-self masks over the flattened rows
    q: np.ndarray           # full-model probability of each node's token given its ancestors (root: nan)
    path: List[int]         # winning path rows, root first, up to the cut (length j + 1)
    j: int                  # accepted nodes on the winning path
    next_token: int
    leaf_accept: List[int]  # accepted length of every leaf's path


def tree_kernel(model: OracleModel, pending: int, T: int, gamma: int, r: float, thresholds, width: int,
                branch: int = 3, accept_mode: int = ACCEPT_THRESHOLD, plan=None) -> TreeKernel:
    """Hardware-friendly tree building and verification (reading D29):
      * drafting (Alg. 1 lines 6-11 with a tree): step s decodes the step-(s-1) nodes with the sparse
        model (each node attends the committed cache [0, T) and its ancestor chain), expands each
        with its top-`branch` tokens of the sparse log-softmax (temperature 1), and keeps the `width`
        candidates of largest cumulative log-likelihood, ties to the lower parent rank then the lower
        token id ("a fixed number of leaves ... through tree pruning based on ranking the cumulative
        log-likelihood of the path"); step 1 keeps the root's top max(width, branch) tokens pruned to
        `width`;
      * verification: one dense forward over all 1 + (gamma-1) width rows with ancestor masks;
      * every leaf's path is scanned like a linear kernel (q = softmax(full logits of the parent
        row)[node token] >= r); the path with the longest accepted prefix wins ("select the one that
        reaches the longest advance length"), ties to the higher leaf cumulative log-likelihood, then
        the lower leaf row; the interleaved token is the full model's argmax at the cut node;
      * the winning path's full-model K/V rows are rewritten into cache slots [T, T+j] (rollback +
        KV rewrite on a tree)."""
    S, W = gamma - 1, width
    n_rows = 1 + S * W
    assert n_rows <= min(64, model.max_gamma), "tree rows must fit the 64-bit masks and the staging area"
    toks, parent, cum, vis = [pending], [-1], [0.0], [1]
    frontier = [0]
    for s in range(1, S + 1):
        cands = []  # (cum, parent rank, token, parent row)
        for pr, f in enumerate(frontier):
            row = model.forward_row(toks[f], T + s - 1, True, thresholds, stage_row=f, plan=plan, tree_vis=vis[f],
                                    tree_n_cache=T)
            lp = log_softmax(row.logits)
            nb = max(W, branch) if s == 1 else branch
            top = np.lexsort((np.arange(lp.size), -lp))[:nb]
            cands += [(cum[f] + float(lp[t]), pr, int(t), f) for t in top]
        keep = sorted(cands, key=lambda c: (-c[0], c[1], c[2]))[:W]
        frontier = []
        for w, (c, pr, t, f) in enumerate(keep):
            n = 1 + (s - 1) * W + w
            toks.append(t)
            parent.append(f)
            cum.append(c)
            vis.append(vis[f] | (1 << n))
            frontier.append(n)
    step = [0] + [1 + (n - 1) // W for n in range(1, n_rows)]
    lf = np.stack([model.forward_row(toks[n], T + step[n], False, None, stage_row=n, tree_vis=vis[n], tree_n_cache=T).logits
                   for n in range(n_rows)])
    q = np.full(n_rows, np.nan)
    for n in range(1, n_rows):
        q[n] = softmax_prob(lf[parent[n]], toks[n])
    best, leaf_acc = None, []
    for w in range(W):
        leaf = 1 + (S - 1) * W + w if S > 0 else 0
        chain = []
        n = leaf
        while n > 0:
            chain.append(n)
            n = parent[n]
        chain.reverse()
        acc = 0
        for n in chain:
            ok = q[n] >= r if accept_mode == ACCEPT_THRESHOLD else toks[n] == argmax_lowest(lf[parent[n]])
            if not ok:
                break
            acc += 1
        leaf_acc.append(acc)
        key = (acc, cum[leaf], -leaf)
        if best is None or key > best[0]:
            best = (key, [0] + chain[:acc])
    path = best[1]
    j = len(path) - 1
    nxt = argmax_lowest(lf[path[-1]])
    model.kv_rewrite_rows(T, path)
    return TreeKernel(toks, parent, cum, vis, q, path, j, nxt, leaf_acc)


@dataclass
class GenerateResult:
    tokens: List[int]
    kernels: List[KernelRecord] = field(default_factory=list)
    all_tokens: List[int] = field(default_factory=list)  # untruncated (includes the last kernel's surplus)
    plan: Optional[np.ndarray] = None  # CSparse neuron plan [L, ffn] when csparse_keep was given

    @property
    def advances(self) -> List[int]:
        return [k.advance for k in self.kernels]

    def rejection_positions(self) -> List[int]:
        """Index i (0-based draft position within the kernel) of every rejected draft: the data of the
        paper's rejection-position histogram (Appendix)."""
        return [k.j for k in self.kernels if k.j < len(k.tokens) - 1]


def generate(model: OracleModel, prompt: Sequence[int], n_tokens: int, gamma: int, r: float,
             thresholds: Optional[np.ndarray], accept_mode: int = ACCEPT_THRESHOLD, rewrite: bool = True,
             interleave: bool = True, rollback: bool = True, csparse_keep: Optional[float] = None,
             tree_width: Optional[int] = None, tree_branch: int = 3, topk_keep: Optional[float] = None,
             temperature: float = 0.0, seed: int = 0) -> GenerateResult:
    """The Sirius loop, Algorithm 1, readings D5-D18:
      * dense prefill of the prompt; the first generated token is the dense argmax (D17);
      * kernel size n = gamma: the sparse model drafts gamma-1 tokens after the pending token,
        writing its K/V at T..T+gamma-2 (Alg. 1 lines 6-11, 'Running sparse model');
      * the full model verifies [pending, d_1..d_{g-1}] at T..T+g-1 in one pass (line 'FORWARD(M_F..)');
      * accept scan with threshold r (lines 12-16); rollback to T+j+1 (line 'cache_pos <- j+1');
      * KV rewrite of the committed span [T, T+j] with the full model's K/V;
      * interleave the full model's argmax of row j (line 'Interleaving Key Token', reading D10/D11).
    Generates exactly n_tokens tokens (D18); the final kernel's surplus is truncated.

    Component ablation (Table 4, §5.3; reading D27): `rewrite`
    (KV Rewrite), `interleave`, `rollback` switch the three correction components independently
    (rollback needs interleave: Table 4 has no rollback without it).  Without rollback every kernel
    commits all gamma positions: the drafts d_1..d_{g-1}, where `interleave` replaces each REJECTED
    draft d_{i+1} (q_i < r) by the full model's argmax of verify row i ("only letting the LLM correct
    the token it is evaluating"), then the full model's token of the last row; with `rewrite` the
    full model's K/V of the g verified rows overwrite the cache rows [T, T+g).  KernelRecord.j stays
    the first rejection (the statistic), the advance is then g.

    csparse_keep: the sparse model is CSparse (Griffin PAPER.md:471) instead of CATS: the
    neuron plan of the prompt (prefill_stats + csparse_plan, reading D28) fixed for the generation.

    tree_width: hardware-friendly tree building and verification (tree_kernel)
    instead of the greedy chain; width 1 is the chain (pinned bitwise).

    topk_keep: the sparse model is top-k FSparse (PAPER.md:121 footnote, reading D30) instead of CATS.

    temperature > 0: every drafted token and every interleaved / bonus token is sampled (sample_token,
    uniform sample_uniform(seed, 0, position of the token)) instead of argmax (reading D31); the
    acceptance q keeps temperature 1."""

    def pick(l, pos):
        return argmax_lowest(l) if temperature <= 0 else sample_token(l, temperature, sample_uniform(seed, 0, pos))
    assert interleave or not rollback, "rollback without interleave is not a Sirius configuration (Table 4)"
    P = len(prompt)
    assert P + n_tokens + gamma <= model.max_seq and gamma >= 1
    # dense prefill; only the last row's logits are needed (prefill_last: same cache, pinned bitwise
    # against prefill() in tests/test_oracle_pins.py)
    plan = None
    if csparse_keep is None:
        out = [argmax_lowest(model.prefill_last(prompt))]  # out[-1] is the pending token at position T
    else:
        lg, stats = model.prefill_stats(prompt)
        plan = csparse_plan(stats, csparse_keep)
        out = [argmax_lowest(lg[-1])]
    T = P
    res = GenerateResult(out)
    res.plan = plan
    topk = None if topk_keep is None else np.full(model.cfg.n_layers, topk_keep, dtype=np.float32)
    while len(out) < n_tokens and tree_width is not None:
        assert rewrite and interleave and rollback, "tree kernels run with every correction component"
        tk = tree_kernel(model, out[-1], T, gamma, r, thresholds, tree_width, tree_branch, accept_mode, plan)
        committed = [tk.tokens[n] for n in tk.path[1:]] + [tk.next_token]
        out += committed
        res.kernels.append(KernelRecord(T, [tk.tokens[n] for n in tk.path], tk.j, tk.q, tk.next_token,
                                        np.zeros((0, model.cfg.n_layers), dtype=np.int32), advance=tk.j + 1, tree=tk))
        T += tk.j + 1
    while len(out) < n_tokens:
        ins = [out[-1]]
        nact, dmarg = [], []
        for i in range(gamma - 1):  # sparse drafting, greedy (D13)
            row = model.decode(ins[i], T + i, True, thresholds, plan=plan, topk=topk)
            nact.append(row.n_active)
            dmarg.append(top2_margin(row.logits) if temperature <= 0 else
                         sample_margin(row.logits, temperature, sample_uniform(seed, 0, T + i + 1)))
            ins.append(pick(row.logits, T + i + 1))
        lf = model.verify(ins, T)  # full model over the kernel, K/V -> staging
        j, q = accept_scan(lf, ins, r, accept_mode)
        if rollback:
            adv = j + 1
            nxt = pick(lf[j], T + j + 1)
            committed = ins[1:j + 1] + [nxt]
        else:  # no rollback: every position is committed; rejected drafts interleaved (or kept)
            adv = gamma
            committed = []
            for i in range(gamma - 1):
                ok = (q[i] >= r) if accept_mode == ACCEPT_THRESHOLD else (ins[i + 1] == argmax_lowest(lf[i]))
                committed.append(ins[i + 1] if (ok or not interleave) else argmax_lowest(lf[i]))
            nxt = argmax_lowest(lf[gamma - 1])
            committed.append(nxt)
        if rewrite:
            model.kv_rewrite(T, adv)  # commit (+ rollback): len = T + adv
        out += committed
        res.kernels.append(KernelRecord(T, list(ins), j, q, nxt,
                                        np.array(nact, dtype=np.int32).reshape(-1, model.cfg.n_layers),
                                        np.array(dmarg), np.array([top2_margin(l) for l in lf]), adv))
        T += adv
    res.all_tokens = list(out)
    res.tokens = out[:n_tokens]
    return res


def greedy_decode(model: OracleModel, prompt: Sequence[int], n_tokens: int, sparse: bool = False,
                  thresholds=None) -> List[int]:
    """Plain autoregressive greedy decode (dense = M_F, or CS-only = M_S) after a dense prefill."""
    logits = model.prefill(prompt)
    out = [argmax_lowest(logits[-1])]
    for i in range(n_tokens - 1):
        row = model.decode(out[-1], len(prompt) + i, sparse, thresholds)
        out.append(argmax_lowest(row.logits))
    return out


# ---------------------------------------------------------------- efficiency formulas (report fields)
def apu(n_sparse: float, c_sparse: float, c_full: float, n_aal: float) -> float:
    """Eq. 1: APU = (n_sparse * C_sparse + C_full) / n_AAL."""
    return (n_sparse * c_sparse + c_full) / n_aal


def effective_density(n_period: float, global_density: float, n_aal: float) -> float:
    """Eq. 3: ((n_period - 1) * I_globalsparsity + 1) / n_AAL."""
    return ((n_period - 1) * global_density + 1) / n_aal


def sd_expected_aal(alpha: float, gamma: int) -> float:
    """§2.3: AAL = (1 - alpha^(gamma+1)) / (1 - alpha)."""
    return (1 - alpha ** (gamma + 1)) / (1 - alpha)


def param_counts(cfg) -> Dict[str, int]:
    """Exact parameter counts by shape arithmetic (untied head); norms counted with attention/head."""
    d, L, hd = cfg.d_model, cfg.n_layers, cfg.head_dim
    attn = L * (d * (cfg.n_heads + 2 * cfg.n_kv_heads) * hd + cfg.n_heads * hd * d + d)
    mlp = L * (3 * d * cfg.ffn_dim + d)
    emb = cfg.vocab * d
    head = cfg.vocab * d + d
    return dict(attention=attn, mlp=mlp, embedding=emb, head=head, total=attn + mlp + emb + head)


def global_density(cfg, keep: float, mode: str) -> float:
    """I_globalsparsity = C_sparse / C_full (Eq. 2).  FSparse sparsifies up+down only
    (PAPER.md:121 'Up and Down linear layers only'); CSparse the whole MLP.  C_full counts every
    parameter (the paper's "MLP ... roughly 70% of the LLM total weights")."""
    c = param_counts(cfg)
    full = c["total"]
    mats = 2 if mode == "fsparse" else 3
    return (full - (1 - keep) * mats * cfg.d_model * cfg.ffn_dim * cfg.n_layers) / full
