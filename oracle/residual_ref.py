"""Canonical residual layouts written out from their definitions — TEST INFRASTRUCTURE ONLY.

BCSR (§3.2, Fig. 2(d)): one segment per vertex holding its in-
and out-neighbours, "sort the column list in ascending order by vertex ID"
(P:325).  Readings: parallel edges are summed;
an antiparallel pair shares one arc pair with cf(u->v) = sum c(u,v) and
cf(v->u) = sum c(v,u); self-loops are dropped; pairs whose capacities
are all zero are KEPT ("cf = 0 arcs are stored, never deleted");
mate[p] = the slot of the reverse arc, i.e. the paper's binary search done once
(P:325-326).

RCSR (Fig. 2(c)): forward CSR of the distinct directed pairs (parallel
edges summed, antiparallel pairs kept distinct) plus a reverse CSR whose entries
hold flow_idx = the forward arc they pair with ("The flow_idx records the index
of backward flow rather than the value").  Both sorted by column.

These are numpy lexsort/unique/searchsorted over the definitions: no blocking,
no fusion; the CUDA build must reproduce them bit-exactly.
"""
from __future__ import annotations

import numpy as np


def _src(n, row_off):
    return np.repeat(np.arange(n, dtype=np.int64), np.diff(np.asarray(row_off, np.int64)))


def bcsr(n, row_off, col, cap):
    """Returns dict(off i64[n+1], col i32[M], cf0 i32[M], mate i32[M])."""
    u = _src(n, row_off)
    v = np.asarray(col, np.int64)
    c = np.asarray(cap, np.int64)
    keep = u != v
    u, v, c = u[keep], v[keep], c[keep]
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    caps = np.concatenate([c, np.zeros_like(c)])
    key = rows * n + cols
    uk, inv = np.unique(key, return_inverse=True)
    cf0 = np.zeros(uk.shape[0], np.int64)
    np.add.at(cf0, inv, caps)
    r = uk // n
    cc = uk % n
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=off[1:])
    mate = np.searchsorted(uk, cc * n + r)
    assert np.array_equal(uk[mate], cc * n + r)
    return dict(off=off, col=cc.astype(np.int32), cf0=cf0, mate=mate.astype(np.int32))


def rcsr(n, row_off, col, cap):
    """Returns dict(foff, fcol, fcf0, roff, rcol, fidx)."""
    u = _src(n, row_off)
    v = np.asarray(col, np.int64)
    c = np.asarray(cap, np.int64)
    keep = u != v
    u, v, c = u[keep], v[keep], c[keep]
    key = u * n + v
    uk, inv = np.unique(key, return_inverse=True)
    fcf0 = np.zeros(uk.shape[0], np.int64)
    np.add.at(fcf0, inv, c)
    fu = uk // n
    fv = uk % n
    foff = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(fu, minlength=n), out=foff[1:])
    # reverse CSR: forward arc i = (fu, fv) appears in fv's reverse segment with column fu
    order = np.lexsort((fu, fv))
    roff = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(fv, minlength=n), out=roff[1:])
    return dict(foff=foff, fcol=fv.astype(np.int32), fcf0=fcf0, roff=roff,
                rcol=fu[order].astype(np.int32), fidx=order.astype(np.int32))
