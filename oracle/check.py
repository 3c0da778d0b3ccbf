"""Validity and certificate checks V1-V7 — TEST INFRASTRUCTURE ONLY.

The same checks run on the oracle's output and on the CUDA path's output.
They prove optimality independently of any oracle: V6 (every S->T edge
saturated, every T->S edge empty) gives F = cap(S, T) and weak duality
(a flow value never exceeds a cut capacity) makes both optimal;
V7 pins S to the canonical S* exactly.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order


class CheckError(AssertionError):
    pass


def _edges(n, row_off):
    return np.repeat(np.arange(n, dtype=np.int64), np.diff(np.asarray(row_off, np.int64)))


def reaches_target(n, src, dst, resid_fwd, resid_bwd, t) -> np.ndarray:
    """bool[n]: v reaches t in G_f, where edge i gives arc src->dst if resid_fwd[i] > 0
    and arc dst->src if resid_bwd[i] > 0.  BFS from t on the reversed residual graph."""
    a_src = np.concatenate([src[resid_fwd > 0], dst[resid_bwd > 0]])
    a_dst = np.concatenate([dst[resid_fwd > 0], src[resid_bwd > 0]])
    # reversed arcs: dst -> src
    R = sp.csr_matrix((np.ones(a_src.shape[0], np.int8), (a_dst, a_src)), shape=(n, n))
    order = breadth_first_order(R, int(t), directed=True, return_predecessors=False)
    out = np.zeros(n, bool)
    out[order] = True
    return out


def check_flow(n, row_off, col, cap, s, t, F, in_S, edge_flow, strict: bool = False):
    """Run V1-V7 on a per-input-edge flow assignment.  Raises CheckError."""
    src = _edges(n, row_off)
    col = np.asarray(col, np.int64)
    cap = np.asarray(cap, np.int64)
    f = np.asarray(edge_flow, np.int64)
    inS = np.asarray(in_S).astype(bool)
    loop = src == col
    # V1 capacity constraints
    if np.any(f < 0) or np.any(f > cap):
        raise CheckError("V1: flow outside [0, c]")
    if np.any(f[loop] != 0):
        raise CheckError("V1: flow on a self-loop")
    # V2 excess / conservation
    exc = np.bincount(col, weights=f, minlength=n) - np.bincount(src, weights=f, minlength=n)
    exc = exc.astype(np.int64)
    others = np.ones(n, bool)
    others[[s, t]] = False
    if np.any(exc[others] < 0):
        raise CheckError("V2: negative excess")
    if strict and np.any(exc[others] != 0):
        raise CheckError("V2(strict): conservation violated")
    # V3
    if int(exc[t]) != int(F):
        raise CheckError(f"V3: excess(t)={int(exc[t])} != F={F}")
    # V4
    if not inS[s] or inS[t]:
        raise CheckError("V4: s must be in S and t outside")
    # V5 stranded excess only on the source side
    if np.any((exc > 0) & others & ~inS):
        raise CheckError("V5: excess outside S")
    # V6 saturation of the cut
    st = inS[src] & ~inS[col]
    ts = ~inS[src] & inS[col]
    if np.any(f[st] != cap[st]):
        raise CheckError("V6: an S->T edge is not saturated")
    if np.any(f[ts] != 0):
        raise CheckError("V6: a T->S edge carries flow")
    if int(cap[st].sum()) != int(F):
        raise CheckError("V6: cut capacity != F")
    # V7 every v outside S reaches t in G_f, and no v in S does
    r = reaches_target(n, src, col, cap - f, f, t)
    if not np.array_equal(r, ~inS):
        raise CheckError("V7: S is not V minus {v reaching t in G_f}")
    return True


def demerge_bcsr(n, row_off, col, cap, off, arc_col, cf, cap0, mate):
    """Per-input-edge flows from a merged BCSR residual state.

    Slot p in seg(u) with column v carries net flow x = cap0[p] - cf[p] from u to v
    (pair conservation cf[p] + cf[mate[p]] = cap0[p] + cap0[mate[p]] is checked here
    too).  x is assigned greedily to the parallel (u, v) input edges in
    input order; reverse (v, u) input edges carry 0 when x >= 0."""
    off = np.asarray(off, np.int64)
    arc_col = np.asarray(arc_col, np.int64)
    cf = np.asarray(cf, np.int64)
    cap0 = np.asarray(cap0, np.int64)
    mate = np.asarray(mate, np.int64)
    M = arc_col.shape[0]
    if np.any(cf < 0):
        raise CheckError("V1(merged): negative residual capacity")
    if M and np.any(cf + cf[mate] != cap0 + cap0[mate]):
        raise CheckError("V1(merged): pair capacity not conserved")
    owner = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    x = cap0 - cf
    key = owner * n + arc_col
    src = _edges(n, row_off)
    col = np.asarray(col, np.int64)
    cap = np.asarray(cap, np.int64)
    f = np.zeros(col.shape[0], np.int64)
    ekey = src * n + col
    pos = np.searchsorted(key, ekey)
    remaining = {}
    for i in range(col.shape[0]):
        u, v = int(src[i]), int(col[i])
        if u == v:
            continue
        p = int(pos[i])
        if p >= M or key[p] != ekey[i]:
            raise CheckError(f"demerge: input edge {i} has no BCSR slot")
        r = remaining.setdefault(p, max(int(x[p]), 0))
        d = min(r, int(cap[i]))
        f[i] = d
        remaining[p] = r - d
    if any(v != 0 for v in remaining.values()):
        raise CheckError("demerge: net flow exceeds the parallel-edge capacities")
    return f


def demerge_rcsr(n, row_off, col, cap, foff, fcol, fcf, cap0, bcf):
    """Per-input-edge flows from an RCSR residual state: forward arc p carries
    flow cap0[p] - fcf[p] (= bcf[p]); assigned greedily to its parallel input edges."""
    foff = np.asarray(foff, np.int64)
    fcol = np.asarray(fcol, np.int64)
    fcf = np.asarray(fcf, np.int64)
    cap0 = np.asarray(cap0, np.int64)
    bcf = np.asarray(bcf, np.int64)
    if np.any(fcf < 0) or np.any(bcf < 0):
        raise CheckError("V1(rcsr): negative residual capacity")
    if np.any(fcf + bcf != cap0):
        raise CheckError("V1(rcsr): forward + backward cf != capacity")
    owner = np.repeat(np.arange(n, dtype=np.int64), np.diff(foff))
    key = owner * n + fcol
    x = cap0 - fcf
    src = _edges(n, row_off)
    col = np.asarray(col, np.int64)
    cap = np.asarray(cap, np.int64)
    f = np.zeros(col.shape[0], np.int64)
    pos = np.searchsorted(key, src * n + col)
    remaining = {}
    for i in range(col.shape[0]):
        if src[i] == col[i]:
            continue
        p = int(pos[i])
        if p >= key.shape[0] or key[p] != src[i] * n + col[i]:
            raise CheckError(f"demerge: input edge {i} has no RCSR arc")
        r = remaining.setdefault(p, int(x[p]))
        d = min(r, int(cap[i]))
        f[i] = d
        remaining[p] = r - d
    if any(v != 0 for v in remaining.values()):
        raise CheckError("demerge: arc flow exceeds its parallel-edge capacities")
    return f
