"""The device pairing's argument (csrc/build.cu "Device restatement of
_pair_to_power_of_two"), checked on the CPU against the literal greedy of
the oracle (bvh.py:98-181 restated): the complete greedy matching of the
path from the local rule (distance to the local minimum of each key run),
the `need` smallest keys of it, and the final-slack test that proves no
deferral happened.  Whenever the test passes the result must equal the
greedy; the device kernels compute exactly these quantities."""

import numpy as np
import pytest

from oracle import meshdist_oracle as oracle


def _rule(sa, n):
    """numpy statement of the device algorithm; None when the device falls
    back to the host greedy (slack could have reached 0)."""
    L = 1 << (n.bit_length() - 1)
    need = n - L
    if need == 0:
        return []
    E = n - 1
    idx = np.arange(E)

    def less(i, j):
        return (sa[i] < sa[j]) | ((sa[i] == sa[j]) & (i < j))

    ls = np.zeros(E, bool)
    ls[1:] = less(idx[:-1], idx[1:])
    rs = np.zeros(E, bool)
    rs[:-1] = less(idx[1:], idx[:-1])
    S = np.maximum.accumulate(np.where(ls, -1, idx))
    Eend = np.minimum.accumulate(np.where(rs, E, idx)[::-1])[::-1]
    m = np.zeros(E, bool)
    m[~ls & ~rs] = True
    a = ls & ~rs
    m[a] = ((idx[a] - S[a]) % 2) == 0
    b = ~ls & rs
    m[b] = ((Eend[b] - idx[b]) % 2) == 0
    c = np.flatnonzero(ls & rs)
    m[c] = (((c - 1 - S[c - 1]) % 2) != 0) & (((Eend[c + 1] - (c + 1)) % 2) != 0)
    cand = np.flatnonzero(m)
    if len(cand) < need or np.isnan(sa).any():
        return None
    order = np.lexsort((cand, sa[cand]))
    lefts = np.sort(cand[order[:need]])
    is_left = np.zeros(n, bool)
    is_left[lefts] = True
    merged = is_left.copy()
    merged[1:] |= is_left[:-1]
    t = np.arange(n)
    start_flag = np.ones(n, bool)
    start_flag[1:] = merged[:-1]
    start = np.maximum.accumulate(np.where(start_flag, t, -1))
    supply = int(np.sum(~merged & (((t - start) % 2) == 1)))
    return list(lefts) if supply >= 1 else None


@pytest.mark.parametrize("seed", range(40))
def test_local_rule_equals_greedy(seed):
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
    got = _rule(sa, n)
    want = oracle.greedy_pairs(sa, n)
    if got is not None:
        assert list(got) == list(want), (seed, n)


def test_local_rule_used_on_most_inputs():
    """The slack test passes on typical inputs (else the device would fall
    back to the host every time)."""
    rng = np.random.default_rng(7)
    passed = 0
    for _ in range(30):
        n = int(rng.integers(100, 5000))
        sa = rng.random(n - 1)
        r = _rule(sa, n)
        if r is not None:
            passed += 1
            assert list(r) == list(oracle.greedy_pairs(sa, n))
    assert passed >= 20
