"""The device pairing's argument (csrc/build.cu "Device restatement of
_pair_to_power_of_two"), checked on the CPU against the literal greedy of
the oracle (bvh.py:98-181 restated).  Phase 1: the complete greedy matching
of the path from the local rule (distance to the local minimum of each key
run), taken in key order while the reference's slack stays positive (a
pick is costly when the run around it at that moment -- bounded by the
nearest smaller-key picks -- has even length and the pick an odd offset).
Phase 2 (slack 0): even runs take their even offsets, odd runs peel their
smallest-key pair.  This numpy model computes exactly what the device
kernels compute; it must equal the greedy on every input."""

import numpy as np
import pytest

from oracle import meshdist_oracle as oracle


def _rule(sa, n):
    """numpy model of the device pairing: phase 1 (unconstrained greedy
    matching prefix while slack > 0), phase 2 (per run: even runs take even
    offsets, odd runs peel their min-key pair)."""
    L = 1 << (n.bit_length() - 1)
    need = n - L
    if need == 0:
        return []
    E = n - 1
    idx = np.arange(E)
    less = lambda i, j: (sa[i] < sa[j]) | ((sa[i] == sa[j]) & (i < j))
    ls = np.zeros(E, bool); ls[1:] = less(idx[:-1], idx[1:])
    rs = np.zeros(E, bool); rs[:-1] = less(idx[1:], idx[:-1])
    S = np.maximum.accumulate(np.where(ls, -1, idx))
    Ee = np.minimum.accumulate(np.where(rs, E, idx)[::-1])[::-1]
    m = np.zeros(E, bool); m[~ls & ~rs] = True
    a = ls & ~rs; m[a] = ((idx[a] - S[a]) % 2) == 0
    b = ~ls & rs; m[b] = ((Ee[b] - idx[b]) % 2) == 0
    c = np.flatnonzero(ls & rs); m[c] = (((c - 1 - S[c - 1]) % 2) != 0) & (((Ee[c + 1] - (c + 1)) % 2) != 0)
    M = np.flatnonzero(m)
    order = np.lexsort((M, sa[M]))  # key rank order of M
    rank = np.empty(len(M), np.int64); rank[order] = np.arange(len(M))
    # nearest smaller (by key) M element on each side (position order)
    left = np.full(len(M), -1); st = []
    for q in range(len(M)):
        while st and rank[st[-1]] > rank[q]: st.pop()
        left[q] = st[-1] if st else -1; st.append(q)
    right = np.full(len(M), -1); st = []
    for q in range(len(M) - 1, -1, -1):
        while st and rank[st[-1]] > rank[q]: st.pop()
        right[q] = st[-1] if st else -1; st.append(q)
    s = np.where(left >= 0, M[np.maximum(left, 0)] + 2, 0)
    e = np.where(right >= 0, M[np.maximum(right, 0)] - 1, n - 1)
    costly = (((e - s + 1) % 2) == 0) & (((M - s) % 2) == 1)
    slack0 = n // 2 - need
    cs = np.cumsum(costly[order])
    hit = np.flatnonzero(slack0 - cs[:need] <= 0)
    if slack0 > 0 and len(hit) == 0:
        return sorted(M[order[:need]].tolist())
    k = hit[0] if slack0 > 0 else -1  # the slack may start at 0: no phase-1 pick at all
    is_left = np.zeros(n, bool); is_left[M[order[:k + 1]]] = True
    merged = is_left.copy(); merged[1:] |= is_left[:-1]
    um = ~merged
    d = np.diff(np.concatenate([[0], um.astype(np.int8), [0]]))
    starts = np.flatnonzero(d == 1); ends = np.flatnonzero(d == -1) - 1
    for s0, e0 in zip(starts, ends):
        ln = e0 - s0 + 1
        if ln < 2:
            continue
        lo, hi = s0, e0
        while hi - lo + 1 >= 2:
            if (hi - lo + 1) % 2 == 0:
                is_left[np.arange(lo, hi, 2)] = True
                break
            seg = np.arange(lo, hi)  # pairs lo .. hi-1
            i = seg[np.lexsort((seg, sa[seg]))[0]]
            is_left[i] = True
            lp = (lo, i - 1); rp = (i + 2, hi)
            # the even part is fully taken, the odd continues
            for (a0, b0) in (lp, rp):
                if b0 - a0 + 1 >= 2 and (b0 - a0 + 1) % 2 == 0:
                    is_left[np.arange(a0, b0, 2)] = True
            lo, hi = lp if (lp[1] - lp[0] + 1) % 2 == 1 else rp
    return sorted(np.flatnonzero(is_left).tolist())


@pytest.mark.parametrize("seed", range(60))
def test_two_phase_rule_equals_greedy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 3000))
    kind = seed % 4
    if kind == 0:
        sa = rng.random(n - 1)
    elif kind == 1:  # heavy ties: index order decides
        sa = rng.integers(0, 3, n - 1).astype(np.float64)
    elif kind == 2:  # long monotone runs
        sa = np.cumsum(rng.random(n - 1)) * (1 if seed % 8 < 4 else -1)
    else:  # all equal (one run rising with the index)
        sa = np.full(n - 1, 0.25)
    assert list(_rule(sa, n)) == list(oracle.greedy_pairs(sa, n)), (seed, n, kind)


@pytest.mark.parametrize("n", range(3, 70))
def test_two_phase_rule_small_n(n):
    """Every small size, where the slack may start at 0 (n = 3, 5, 6, 7,
    11, ...): random, tied and monotone keys."""
    rng = np.random.default_rng(n)
    for sa in (rng.random(n - 1), rng.integers(0, 2, n - 1).astype(np.float64), np.arange(n - 1, 0, -1.0),
               np.full(n - 1, 1.0)):
        assert list(_rule(sa, n)) == list(oracle.greedy_pairs(sa, n)), (n, sa)


def test_two_phase_rule_on_torus_pairing():
    """A torus (the rings' geometry, where the slack reaches 0 and phase 2
    decides most merges): the model equals the literal greedy."""
    from paper_2411_11244_b200 import scenes

    tz, _ = scenes.ring_pair_base(120, 45)
    V, T = np.asarray(tz.vertices), np.asarray(tz.triangles)
    _, order = oracle.morton_order(V, T)
    P = V[T]
    sa = oracle.pair_surface_areas(order, P.min(axis=1), P.max(axis=1))
    assert list(_rule(sa, len(T))) == list(oracle.greedy_pairs(sa, len(T)))
