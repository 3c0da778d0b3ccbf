"""Brute-force pins for the oracle — TEST INFRASTRUCTURE ONLY.

edmonds_karp(): BFS augmenting paths (§2.1, "Edmonds and Karp
improved the efficiency of finding augmenting paths using breadth-first search").
enum_mincut():  exhaustive enumeration of every s-t cut of a tiny graph; the
minimum is F* by max-flow/min-cut duality (P:120-127 defines both problems).
Both are plain pure-Python loops for tiny inputs only (n <= ~16).
"""
from __future__ import annotations

from collections import deque
from typing import Tuple

import numpy as np


def _cap_matrix(n, row_off, col, cap):
    C = [[0] * n for _ in range(n)]
    for u in range(n):
        for i in range(int(row_off[u]), int(row_off[u + 1])):
            v = int(col[i])
            if u != v:
                C[u][v] += int(cap[i])
    return C


def edmonds_karp(n, row_off, col, cap, s, t) -> int:
    """Max-flow value by shortest augmenting paths on the summed capacity matrix."""
    C = _cap_matrix(n, row_off, col, cap)
    F = [[0] * n for _ in range(n)]
    total = 0
    while True:
        par = [-1] * n
        par[s] = s
        q = deque([s])
        while q and par[t] < 0:
            u = q.popleft()
            for v in range(n):
                if par[v] < 0 and C[u][v] - F[u][v] > 0:
                    par[v] = u
                    q.append(v)
        if par[t] < 0:
            return total
        # bottleneck
        d = None
        v = t
        while v != s:
            u = par[v]
            r = C[u][v] - F[u][v]
            d = r if d is None else min(d, r)
            v = u
        v = t
        while v != s:
            u = par[v]
            F[u][v] += d
            F[v][u] -= d
            v = u
        total += d


def enum_mincut(n, row_off, col, cap, s, t) -> Tuple[int, np.ndarray]:
    """(min cut capacity, S_max) where S_max is the union of the source sides of
    all minimum cuts (equal to V minus the vertices that reach t in G_f of any
    maximum flow).  Enumerates all 2^(n-2) cuts."""
    src = np.repeat(np.arange(n), np.diff(row_off))
    others = [v for v in range(n) if v not in (s, t)]
    best = None
    union = np.zeros(n, bool)
    for mask in range(1 << len(others)):
        inS = np.zeros(n, bool)
        inS[s] = True
        for j, v in enumerate(others):
            if mask >> j & 1:
                inS[v] = True
        c = int(cap[(inS[src]) & (~inS[col])].sum())
        if best is None or c < best:
            best = c
            union = inS.copy()
        elif c == best:
            union |= inS
    return best, union.astype(np.uint8)
