"""Pins for the oracle's tree building and verification (§4.3;
reading D29): each part is checked against sequential decoding of single paths with a fresh model
(no staging area, no ancestor masks, no pruning code) or against the linear chain.  CPU only."""
import numpy as np
import pytest

import synth
from oracle import sirius_oracle as so

GAMMA = 4


@pytest.fixture(scope="module")
def setup(tiny):
    cfg, w = tiny
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 7, 40)
    return cfg, w, thr, prompt


def _fresh(cfg, w, prompt):
    m = so.OracleModel(cfg, w, max_seq=128, max_gamma=64)
    lg = m.prefill(prompt)
    return m, so.argmax_lowest(lg[-1])


def _path(tk, n):
    out = []
    while n > 0:
        out.append(n)
        n = tk.parent[n]
    return out[::-1]


def _seq_logits(cfg, w, prompt, tokens, sparse, thr):
    """Sequential decode of `tokens` (pending first) after the prompt with a fresh model: logits of
    every row — the path written out as an ordinary autoregressive decode."""
    m = so.OracleModel(cfg, w, max_seq=128, max_gamma=64)
    m.prefill(prompt)
    return [m.decode(t, len(prompt) + i, sparse, thr).logits for i, t in enumerate(tokens)]


@pytest.mark.parametrize("r,mode", [(0.1, so.ACCEPT_THRESHOLD), (0.3, so.ACCEPT_THRESHOLD),
                                    (0.0, so.ACCEPT_EXACT_ARGMAX)])
def test_width_one_is_the_linear_chain(setup, r, mode):
    """Degeneracy: tree width 1 reproduces the greedy-chain Sirius loop bit for bit."""
    cfg, w, thr, prompt = setup
    a = so.generate(so.OracleModel(cfg, w, max_seq=128, max_gamma=64), prompt, 24, GAMMA, r, thr, accept_mode=mode)
    b = so.generate(so.OracleModel(cfg, w, max_seq=128, max_gamma=64), prompt, 24, GAMMA, r, thr, accept_mode=mode,
                    tree_width=1)
    assert a.tokens == b.tokens and a.advances == b.advances


@pytest.mark.parametrize("width", [2, 3])
def test_tree_against_sequential_paths(setup, width):
    """Fixed shape; the draft pruning equals a brute-force beam over sequentially decoded paths; every
    node's verify logits equal a sequential dense decode of its root path; every leaf's accepted
    length and the verdict follow from those; the commit equals a dense prefill of the winner."""
    cfg, w, thr, prompt = setup
    m, pending = _fresh(cfg, w, prompt)
    T, S, r, b = len(prompt), GAMMA - 1, 0.3, 3
    tk = so.tree_kernel(m, pending, T, GAMMA, r, thr, width, b)
    n_rows = 1 + S * width
    assert len(tk.tokens) == n_rows and all(0 <= tk.parent[n] < n for n in range(1, n_rows))
    assert all(1 + (tk.parent[n] - 1) // width == (n - 1) // width for n in range(1 + width, n_rows))
    # brute-force beam: log-probs from sequential sparse decodes of each kept node's path
    frontier = [0]
    for s in range(1, S + 1):
        cands = []
        for pr, f in enumerate(frontier):
            path = [0] + _path(tk, f)
            lg = _seq_logits(cfg, w, prompt, [tk.tokens[n] for n in path], True, thr)[-1]
            lp = lg - (lg.max() + np.log(np.exp(lg - lg.max()).sum()))
            for t in range(cfg.vocab):
                cands.append((tk.cum[f] + lp[t], pr, t))
        cands.sort(key=lambda c: (-c[0], c[1], c[2]))
        rows = list(range(1 + (s - 1) * width, 1 + s * width))
        assert [tk.tokens[n] for n in rows] == [c[2] for c in cands[:width]]
        np.testing.assert_allclose([tk.cum[n] for n in rows], [c[0] for c in cands[:width]], rtol=0, atol=1e-12)
        frontier = rows
    # verify rows = sequential dense decode of each root path; q and accepted lengths
    accs = []
    for wl in range(width):
        leaf = 1 + (S - 1) * width + wl
        path = [0] + _path(tk, leaf)
        lg = _seq_logits(cfg, w, prompt, [tk.tokens[n] for n in path], False, None)
        acc = 0
        for i in range(1, len(path)):
            q = so.softmax_prob(lg[i - 1], tk.tokens[path[i]])
            assert abs(q - tk.q[path[i]]) <= 1e-12
            if q < r:
                break
            acc += 1
        accs.append(acc)
    assert accs == tk.leaf_accept
    best = max(range(width), key=lambda wl: (accs[wl], tk.cum[1 + (S - 1) * width + wl], -wl))
    leaf = 1 + (S - 1) * width + best
    assert tk.path == ([0] + _path(tk, leaf))[:accs[best] + 1] and tk.j == accs[best]
    lg = _seq_logits(cfg, w, prompt, [tk.tokens[n] for n in tk.path], False, None)
    assert tk.next_token == so.argmax_lowest(lg[-1])
    # commit: cache [T, T + j] equals a dense prefill of the committed tokens
    ref = so.OracleModel(cfg, w, max_seq=128, max_gamma=64)
    ref.prefill(list(prompt) + [tk.tokens[n] for n in tk.path])
    for l in range(cfg.n_layers):
        k1, v1 = m.read_cache(l, T + tk.j + 1)
        k2, v2 = ref.read_cache(l, T + tk.j + 1)
        np.testing.assert_array_equal(k1, k2)
        np.testing.assert_array_equal(v1, v2)


def test_tree_r0_takes_the_most_likely_full_path(setup):
    """r = 0 accepts every node: every leaf's path is fully accepted, the winner is the leaf of highest
    cumulative log-likelihood, the advance is gamma."""
    cfg, w, thr, prompt = setup
    m, pending = _fresh(cfg, w, prompt)
    tk = so.tree_kernel(m, pending, len(prompt), GAMMA, 0.0, thr, 3)
    S = GAMMA - 1
    assert tk.leaf_accept == [S] * 3 and tk.j == S
    leaves = [1 + (S - 1) * 3 + i for i in range(3)]
    assert tk.path[-1] == max(leaves, key=lambda n: (tk.cum[n], -n))


def test_tree_generate_accounting(setup):
    """Tree Sirius loop: exactly n tokens, advances in [1, gamma] summing to the committed count, and
    a wider tree never accepts fewer tokens on the first kernel than its own greedy chain would."""
    cfg, w, thr, prompt = setup
    res = so.generate(so.OracleModel(cfg, w, max_seq=128, max_gamma=64), prompt, 24, GAMMA, 0.3, thr, tree_width=3)
    assert len(res.tokens) == 24 and all(1 <= a <= GAMMA for a in res.advances)
    assert sum(res.advances) + 1 >= 24
