"""Pins for the reference residual layouts (oracle/residual_ref.py) and for the
validity checker itself (oracle/check.py): worked examples from SPEC.md,
invariants that hold by definition, and mutation tests showing each check
fires on the corruption it exists for."""
import numpy as np
import pytest

import oracle
import synth
from oracle import check, residual_ref


def _g(n, edges, s=0, t=None):
    e = np.array(edges, np.int64).reshape(-1, 3)
    return synth.from_edges(n, e[:, 0], e[:, 1], e[:, 2], s, n - 1 if t is None else t)


def test_bcsr_spec_examples(golden):
    for ex in golden["bcsr"]:
        g = _g(ex["n"], ex["edges"])
        b = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
        for v, seg in ex["segments"].items():
            v = int(v)
            lo, hi = b["off"][v], b["off"][v + 1]
            got = [[int(c), int(f)] for c, f in zip(b["col"][lo:hi], b["cf0"][lo:hi])]
            assert got == seg, ex["citation"]


def test_csr_spec_examples(golden):
    for ex in golden["csr"]:
        g = _g(ex["n"], ex["edges"])
        r = residual_ref.rcsr(g.n, g.row_off, g.col, g.cap)
        if "offsets" in ex:
            assert r["foff"].tolist() == ex["offsets"], ex["citation"]
            assert r["fcol"].tolist() == ex["cols"]
            assert r["fcf0"].tolist() == ex["cf"]
        if "rev_offsets" in ex:
            assert r["roff"].tolist() == ex["rev_offsets"], ex["citation"]
            assert r["rcol"].tolist() == ex["rev_cols"]


def test_star_backward_arc():
    # star centre 0 with leaves 1..8: the backward arc of (5,0) is column 5 in 0's segment
    g = _g(9, [(0, k, 1) for k in range(1, 9)])
    b = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
    p = b["off"][5]                      # leaf 5 has one slot (col 0)
    q = b["mate"][p]
    assert b["col"][q] == 5 and b["off"][0] <= q < b["off"][1]
    # linear scan agrees with the mate index for every slot
    for p in range(b["col"].shape[0]):
        u = int(np.searchsorted(b["off"], p, side="right") - 1)
        v = int(b["col"][p])
        lo, hi = b["off"][v], b["off"][v + 1]
        assert list(b["col"][lo:hi]).index(u) + lo == b["mate"][p]


@pytest.mark.parametrize("seed", range(6))
def test_layout_invariants(seed):
    g = synth.tiny_random(40, 300, 9, seed)
    b = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
    M = b["col"].shape[0]
    mate = b["mate"].astype(np.int64)
    assert np.all(mate[mate] == np.arange(M))           # involution
    assert np.all(mate != np.arange(M))                  # no fixed points
    owner = np.repeat(np.arange(g.n), np.diff(b["off"]))
    assert np.all(b["col"][mate] == owner)
    for v in range(g.n):                                 # strictly sorted segments
        seg = b["col"][b["off"][v]:b["off"][v + 1]]
        assert np.all(np.diff(seg) > 0)
    # total capacity is preserved: sum cf0 == sum of non-self-loop caps
    src, dst, cap = g.edges()
    assert b["cf0"].sum() == cap[src != dst].sum()
    r = residual_ref.rcsr(g.n, g.row_off, g.col, g.cap)
    # representation equivalence: same (neighbour -> total cf) per vertex at construction
    for v in range(g.n):
        fw = dict(zip(r["fcol"][r["foff"][v]:r["foff"][v + 1]].tolist(),
                      r["fcf0"][r["foff"][v]:r["foff"][v + 1]].tolist()))
        nb = dict()
        for c, f in fw.items():
            nb[c] = nb.get(c, 0) + f
        for q in range(r["roff"][v], r["roff"][v + 1]):
            nb[int(r["rcol"][q])] = nb.get(int(r["rcol"][q]), 0) + 0
        bb = dict(zip(b["col"][b["off"][v]:b["off"][v + 1]].tolist(), b["cf0"][b["off"][v]:b["off"][v + 1]].tolist()))
        assert nb == bb
    # flow_idx pairs each reverse entry with its forward arc
    fu = np.repeat(np.arange(g.n), np.diff(r["foff"]))
    rv = np.repeat(np.arange(g.n), np.diff(r["roff"]))
    assert np.all(fu[r["fidx"]] == r["rcol"]) and np.all(r["fcol"][r["fidx"]] == rv)


def test_memory_linearity():
    # cells <= 8 (n + m) for both layouts at n = 1e5, m = 1e6
    n, m = 100_000, 1_000_000
    g = synth.random_graph(n, m, 3)
    b = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
    r = residual_ref.rcsr(g.n, g.row_off, g.col, g.cap)
    M = b["col"].shape[0]
    assert (n + 1) + 3 * M <= 8 * (n + m)            # off + {col, cf, mate}
    mf = r["fcol"].shape[0]
    assert 2 * (n + 1) + 5 * mf <= 8 * (n + m)       # foff, roff + {fcol, fcf, rcol, fidx, bcf}


# ------------------------------------------------------------------ checker mutation tests
def _solved(seed=2):
    g = synth.random_graph(200, 1500, seed, 0, 199)
    return g, oracle.maxflow_graph(g)


def test_checker_accepts_oracle():
    g, r = _solved()
    assert check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


def test_checker_rejects_corruptions():
    g, r = _solved()
    args = (g.n, g.row_off, g.col, g.cap, g.s, g.t)
    f = r.edge_flow.copy()
    i = int(np.argmax(f))
    bad = f.copy(); bad[i] = g.cap[i] + 1
    with pytest.raises(check.CheckError, match="V1"):
        check.check_flow(*args, r.flow, r.in_S, bad)
    bad = f.copy(); bad[i] -= 1
    with pytest.raises(check.CheckError):
        check.check_flow(*args, r.flow, r.in_S, bad, strict=True)
    with pytest.raises(check.CheckError, match="V3"):
        check.check_flow(*args, r.flow + 1, r.in_S, f)
    S = r.in_S.copy(); S[g.t] = 1
    with pytest.raises(check.CheckError, match="V4"):
        check.check_flow(*args, r.flow, S, f)
    # moving a T-side vertex into S breaks V6 or V7
    tv = int(np.nonzero(r.in_S == 0)[0][0] if r.in_S[0] == 0 else [v for v in range(g.n) if not r.in_S[v] and v != g.t][0])
    S = r.in_S.copy(); S[tv] = 1
    with pytest.raises(check.CheckError):
        check.check_flow(*args, r.flow, S, f)


def test_demerge_roundtrip():
    # a strict oracle flow pushed through the merged layout and de-merged again is valid
    g = synth.tiny_random(30, 200, 9, 4, self_loops=True)
    r = oracle.maxflow_graph(g)
    b = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
    owner = np.repeat(np.arange(g.n), np.diff(b["off"]))
    key = owner * g.n + b["col"]
    src, dst, _ = g.edges()
    net = np.zeros(key.shape[0], np.int64)
    keep = src != dst
    np.add.at(net, np.searchsorted(key, src[keep] * g.n + dst[keep]), r.edge_flow[keep])
    x = net - net[b["mate"]]                      # net flow u->v on each slot
    cf = b["cf0"] - x
    f = check.demerge_bcsr(g.n, g.row_off, g.col, g.cap, b["off"], b["col"], cf, b["cf0"], b["mate"])
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, f, strict=True)


def test_demerge_rcsr_roundtrip():
    # the RCSR analogue: a strict oracle flow written into the forward / backward residual
    # capacities of the reference RCSR and de-merged again is valid (V1-V7 strict);
    # antiparallel input edges stay distinct forward arcs in RCSR, so each arc carries only
    # its own direction's flow: fcf = cap0 - f, bcf = f
    g = synth.tiny_random(30, 200, 9, 5, self_loops=True)
    r = oracle.maxflow_graph(g)
    R = residual_ref.rcsr(g.n, g.row_off, g.col, g.cap)
    owner = np.repeat(np.arange(g.n), np.diff(R["foff"]))
    key = owner * g.n + R["fcol"]
    src, dst, _ = g.edges()
    keep = src != dst
    fl = np.zeros(key.shape[0], np.int64)
    np.add.at(fl, np.searchsorted(key, src[keep] * g.n + dst[keep]), r.edge_flow[keep])
    fcf, bcf = R["fcf0"] - fl, fl
    f = check.demerge_rcsr(g.n, g.row_off, g.col, g.cap, R["foff"], R["fcol"], fcf, R["fcf0"], bcf)
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, f, strict=True)
    # per parallel-edge group the de-merged flows sum to the arc flow
    grp = np.searchsorted(key, src[keep] * g.n + dst[keep])
    assert np.array_equal(np.bincount(grp, weights=f[keep], minlength=key.shape[0]).astype(np.int64), fl)
    # corruptions are rejected: capacity not conserved, negative cf
    bad = bcf.copy(); bad[int(np.argmax(bcf))] += 1
    with pytest.raises(check.CheckError):
        check.demerge_rcsr(g.n, g.row_off, g.col, g.cap, R["foff"], R["fcol"], fcf, R["fcf0"], bad)
    bad = fcf.copy(); bad[int(np.argmin(fcf))] = -1
    with pytest.raises(check.CheckError):
        check.demerge_rcsr(g.n, g.row_off, g.col, g.cap, R["foff"], R["fcol"], bad, R["fcf0"], bcf - 0)


def test_check_matching_rejects_mutations():
    # matching validity: each pair an input edge, each l / r at most once, size
    import synth as _s
    from oracle import matching
    nL, nR = 40, 30
    l, r = _s.bipartite_edges(nL, nR, 120, 3)
    n, src, dst, cap, s, t = matching.network(nL, nR, l, r)
    g = _s.from_edges(n, src, dst, cap, s, t)
    res = oracle.maxflow_graph(g)
    # a matching from the oracle's strict flow: left l matched to r when the unit on (1+l, 1+nL+r) flows
    gs, gd, _ = g.edges()
    m = np.full(nL, -1, np.int64)
    for i in np.nonzero(res.edge_flow > 0)[0]:
        if 1 <= gs[i] <= nL and nL + 1 <= gd[i] <= nL + nR:
            m[gs[i] - 1] = gd[i] - 1 - nL
    assert matching.check_matching(nL, nR, l, r, m, res.flow)
    with pytest.raises(AssertionError, match="expected"):
        matching.check_matching(nL, nR, l, r, m, res.flow + 1)
    li = int(np.nonzero(m >= 0)[0][0])
    lj = int(np.nonzero(m >= 0)[0][1])
    bad = m.copy(); bad[lj] = bad[li]                                   # right vertex used twice
    with pytest.raises(AssertionError, match="twice"):
        matching.check_matching(nL, nR, l, r, bad, res.flow)
    edges = set(zip(l.tolist(), r.tolist()))
    rr = next(x for x in range(nR) if (li, x) not in edges and x not in set(m.tolist()))
    bad = m.copy(); bad[li] = rr                                        # not an input edge
    with pytest.raises(AssertionError, match="not an input edge"):
        matching.check_matching(nL, nR, l, r, bad, res.flow)
    bad = m.copy(); bad[li] = nR                                        # out of range
    with pytest.raises(AssertionError, match="out of range"):
        matching.check_matching(nL, nR, l, r, bad, res.flow)
