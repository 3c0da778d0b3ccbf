"""Bipartite matching as max flow — TEST INFRASTRUCTURE ONLY.

Network per PAPER.md §4.1 P:433 ("the super-source and super-sink connect to two
groups of vertices") with the ids of SPEC S:304: s = 0, left l -> 1 + l,
right r -> 1 + nL + r, t = nL + nR + 1, unit capacities.
"""
from __future__ import annotations

import numpy as np


def network(nL, nR, l, r):
    """(n, src, dst, cap, s, t) of the unit-capacity matching network."""
    l = np.asarray(l, np.int64)
    r = np.asarray(r, np.int64)
    n = nL + nR + 2
    s, t = 0, nL + nR + 1
    src = np.concatenate([np.zeros(nL, np.int64), 1 + l, 1 + nL + np.arange(nR)])
    dst = np.concatenate([1 + np.arange(nL), 1 + nL + r, np.full(nR, t)])
    cap = np.ones(src.shape[0], np.int32)
    return n, src, dst, cap, s, t


def check_matching(nL, nR, l, r, match_of_left, size):
    """A valid matching: every pair is an input edge, each l and r used at most once,
    and the number of pairs equals `size`."""
    m = np.asarray(match_of_left, np.int64)
    assert m.shape[0] == nL
    used = m[m >= 0]
    assert np.all(used < nR), "right id out of range"
    assert np.unique(used).shape[0] == used.shape[0], "a right vertex is matched twice"
    assert used.shape[0] == size, f"matching has {used.shape[0]} pairs, expected {size}"
    # every pair is an input edge: membership of l * nR + r in the sorted edge keys
    keys = np.unique(np.asarray(l, np.int64) * nR + np.asarray(r, np.int64))
    li = np.nonzero(m >= 0)[0]
    q = li * nR + m[li]
    pos = np.minimum(np.searchsorted(keys, q), max(keys.shape[0] - 1, 0))
    hit = keys[pos] == q if keys.shape[0] else np.zeros(q.shape[0], bool)
    if not np.all(hit):
        j = int(li[np.nonzero(~hit)[0][0]])
        raise AssertionError(f"pair ({j},{int(m[j])}) is not an input edge")
    return True
