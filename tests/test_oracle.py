"""Pins for the CPU oracle (no GPU): the oracle is checked against things other
than itself — printed worked examples (tests/golden, cited), brute force,
closed forms, library routines and metamorphic relations — chosen so a dropped
term, wrong sign/index or transposed operand fails at least one of them."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import maximum_bipartite_matching, maximum_flow

import oracle
import synth
from oracle import brute, check, matching

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def _g(n, edges, s, t):
    e = np.array(edges, np.int64).reshape(-1, 3)
    return synth.from_edges(n, e[:, 0], e[:, 1], e[:, 2], s, t)


def _scipy_flow(g):
    src, dst, cap = g.edges()
    keep = src != dst
    A = sp.csr_matrix((cap[keep].astype(np.int32), (src[keep], dst[keep])), shape=(g.n, g.n))
    A.sum_duplicates()
    return int(maximum_flow(A, g.s, g.t, method="dinic").flow_value)


# ------------------------------------------------------------------ golden examples
def test_spec_maxflow_examples(golden):
    for ex in golden["maxflow"]:
        g = _g(ex["n"], ex["edges"], ex["s"], ex["t"])
        for gr in (True, False):
            r = oracle.maxflow_graph(g, gr=gr)
            assert r.flow == ex["flow"], (ex["name"], ex["citation"])
            assert r.cut_capacity == ex["flow"]
            check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


def test_spec_preflow_example(golden):
    for ex in golden["preflow"]:
        g = _g(ex["n"], ex["edges"], ex["s"], ex["t"])
        e, tot, _, _ = oracle.initial_state(g.n, g.row_off, g.col, g.cap, g.s, g.t)
        for v, x in ex["excess"].items():
            assert e[int(v)] == x, ex["citation"]
        assert tot == ex["excess_total"]


@pytest.mark.parametrize("seed", range(12))
def test_initial_state_vs_closed_form_and_library_bfs(seed):
    """oracle.initial_state (Alg. 1 Step 0, then one reverse BFS from t)
    against its closed form: e(v) = sum of c(s,v) over edges s->v (self-loops excluded),
    Excess_total = their sum, and level = scipy's unweighted shortest-path distance to t on the
    residual graph after the preflow (every arc out of s saturated, the reverse arcs v->s
    holding c(s,v)); unreached vertices and s itself get n.  The CUDA path's first GR is
    compared with these values bit-exactly (tests/test_gpu_state.py)."""
    from scipy.sparse.csgraph import shortest_path
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(3, 40))
    g = synth.tiny_random(n, int(rng.integers(0, 6 * n)), int(rng.integers(1, 9)), seed)
    e, tot, lv, _ = oracle.initial_state(g.n, g.row_off, g.col, g.cap, g.s, g.t)
    src, dst, cap = g.edges()
    src = src.astype(np.int64); dst = dst.astype(np.int64); cap = cap.astype(np.int64)
    keep = src != dst
    src, dst, cap = src[keep], dst[keep], cap[keep]
    from_s = src == g.s
    want_e = np.bincount(dst[from_s], weights=cap[from_s], minlength=g.n).astype(np.int64)
    want_e[g.s] = 0
    assert np.array_equal(e, want_e) and tot == int(cap[from_s].sum())
    # residual arcs after the preflow: forward u->v with c>0 unless u = s; backward v->u with
    # the flow on (u,v), i.e. c(s,v) when u = s
    fwd = (cap > 0) & ~from_s
    bwd = from_s & (cap > 0)
    a_src = np.concatenate([src[fwd], dst[bwd]])
    a_dst = np.concatenate([dst[fwd], src[bwd]])
    # distances TO t: BFS from t over reversed arcs; s is never expanded
    keep2 = a_dst != g.s   # a reversed arc out of s (an arc into s) would expand s
    R = sp.csr_matrix((np.ones(int(keep2.sum())), (a_dst[keep2], a_src[keep2])), shape=(g.n, g.n))
    d = shortest_path(R, method="D", unweighted=True, indices=g.t)
    want = np.where(np.isinf(d), g.n, d).astype(np.int64)
    want[g.s] = g.n
    assert np.array_equal(lv, want)


def test_spec_global_relabel_example(golden):
    for ex in golden["global_relabel"]:
        g = _g(ex["n"], ex["edges"], ex["s"], ex["t"])
        _, _, _, lv0 = oracle.initial_state(g.n, g.row_off, g.col, g.cap, g.s, g.t)
        for v, h in ex["heights_before_preflow"].items():
            # S:215 gives h(s) = n for s; the BFS reaches s at distance 2 on this path,
            # but the source's label is pinned to |V| by the paper.
            if int(v) == g.s:
                continue
            assert lv0[int(v)] == h, ex["citation"]


def test_spec_matching_examples(golden):
    for ex in golden["matching"]:
        l = np.array([e[0] for e in ex["edges"]], np.int64)
        r = np.array([e[1] for e in ex["edges"]], np.int64)
        n, src, dst, cap, s, t = matching.network(ex["nL"], ex["nR"], l, r)
        g = synth.from_edges(n, src, dst, cap, s, t)
        assert oracle.maxflow_graph(g).flow == ex["size"], ex["citation"]


# ------------------------------------------------------------------ brute force
@pytest.mark.parametrize("seed", range(0, 400))
def test_brute_force_tiny(seed):
    rng = np.random.default_rng(10_000 + seed)
    n = int(rng.integers(2, 11))
    m = int(rng.integers(0, 30))
    g = synth.tiny_random(n, m, int(rng.integers(1, 9)), seed)
    ek = brute.edmonds_karp(g.n, g.row_off, g.col, g.cap, g.s, g.t)
    cut, S_max = brute.enum_mincut(g.n, g.row_off, g.col, g.cap, g.s, g.t)
    assert ek == cut
    for gr, gap in ((True, True), (False, True), (True, False), (False, False)):
        r = oracle.maxflow_graph(g, gr=gr, gap=gap)
        assert r.flow == ek
        assert r.cut_capacity == ek
        assert np.array_equal(r.in_S, S_max)  # canonical S* = union of min-cut source sides (E7)
        check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("k", [2, 8, 33, 128])
def test_unit_grid_closed_form(k):
    # k x k unit grid, S -> column 0, column k-1 -> T: the k row paths are disjoint and a
    # vertical cut has k unit arcs, so F = k (SURVEY §8(c) "What pins each part").
    g = synth.grid(k, k, random_caps=False)
    r = oracle.maxflow_graph(g)
    assert r.flow == k
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


def test_disjoint_paths_closed_form():
    rng = np.random.default_rng(5)
    edges, expect = [], 0
    n = 2
    for _ in range(20):
        L = int(rng.integers(1, 6))
        caps = rng.integers(1, 50, size=L + 1)
        verts = [0] + list(range(n, n + L)) + [1]
        n += L
        for a, b, c in zip(verts[:-1], verts[1:], caps):
            edges.append((a, b, int(c)))
        expect += int(caps.min())
    g = _g(n, edges, 0, 1)
    assert oracle.maxflow_graph(g).flow == expect


@pytest.mark.parametrize("a,b", [(1, 1), (3, 5), (7, 2), (16, 16)])
def test_complete_bipartite_matching(a, b):
    l = np.repeat(np.arange(a), b)
    r = np.tile(np.arange(b), a)
    n, src, dst, cap, s, t = matching.network(a, b, l, r)
    assert oracle.maxflow_graph(synth.from_edges(n, src, dst, cap, s, t)).flow == min(a, b)


def test_unreachable_sink_and_sourceless():
    g = _g(5, [(0, 1, 3), (1, 2, 4), (3, 4, 9)], 0, 4)
    r = oracle.maxflow_graph(g)
    assert r.flow == 0 and r.cut_capacity == 0
    assert list(r.in_S) == [1, 1, 1, 0, 0]   # only 3 and 4 reach t
    g = _g(3, [(1, 2, 4), (2, 0, 3)], 0, 2)
    assert oracle.maxflow_graph(g).flow == 0


# ------------------------------------------------------------------ library routines
@pytest.mark.parametrize("seed", range(1, 17))
def test_c1_vs_scipy_dinic(seed):
    g = synth.random_graph(1024, 8192, seed)
    r = oracle.maxflow_graph(g)
    assert r.flow == _scipy_flow(g) == r.cut_capacity
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


@pytest.mark.parametrize("shape", [(64, 64, True, 3), (40, 90, True, 4)])
def test_random_grid_vs_scipy(shape):
    W, H, rc, seed = shape
    g = synth.grid(W, H, rc, seed)
    r = oracle.maxflow_graph(g)
    assert r.flow == _scipy_flow(g)
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


@pytest.mark.parametrize("rule", ["paper", "hub20"])
def test_rmat_vs_scipy(rule):
    g = synth.rmat(12, 16, 3, rule)
    r = oracle.maxflow_graph(g)
    assert r.flow == _scipy_flow(g)
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)


@pytest.mark.parametrize("seed", range(3))
def test_bipartite_vs_hopcroft_karp(seed):
    nL, nR = 3000, 2500
    l, r = synth.bipartite_edges(nL, nR, 6000, seed)
    n, src, dst, cap, s, t = matching.network(nL, nR, l, r)
    F = oracle.maxflow_graph(synth.from_edges(n, src, dst, cap, s, t)).flow
    B = sp.csr_matrix((np.ones(len(l), np.int8), (l, r)), shape=(nL, nR))
    hk = int((maximum_bipartite_matching(B, perm_type="column") >= 0).sum())
    assert F == hk


# ------------------------------------------------------------------ metamorphic relations
def _rand_instance(seed):
    return synth.random_graph(300, 2400, seed, s=0, t=299)


@pytest.mark.parametrize("seed", range(4))
def test_metamorphic_permutation(seed):
    g = _rand_instance(seed)
    r = oracle.maxflow_graph(g)
    perm = np.random.default_rng(seed).permutation(g.n)
    src, dst, cap = g.edges()
    h = synth.from_edges(g.n, perm[src], perm[dst], cap, perm[g.s], perm[g.t])
    q = oracle.maxflow_graph(h)
    assert q.flow == r.flow
    assert np.array_equal(q.in_S[perm], r.in_S)


@pytest.mark.parametrize("seed", range(4))
def test_metamorphic_reversal(seed):
    g = _rand_instance(seed)
    src, dst, cap = g.edges()
    h = synth.from_edges(g.n, dst, src, cap, g.t, g.s)
    assert oracle.maxflow_graph(h).flow == oracle.maxflow_graph(g).flow


@pytest.mark.parametrize("k", [2, 7])
def test_metamorphic_scaling(k):
    g = _rand_instance(11)
    h = synth.Graph(g.n, g.row_off, g.col, (g.cap * k).astype(np.int32), g.s, g.t)
    r, q = oracle.maxflow_graph(g), oracle.maxflow_graph(h)
    assert q.flow == k * r.flow
    assert np.array_equal(q.in_S, r.in_S)


@pytest.mark.parametrize("seed", range(4))
def test_metamorphic_split_zero_selfloop(seed):
    g = _rand_instance(seed)
    r = oracle.maxflow_graph(g)
    rng = np.random.default_rng(seed)
    src, dst, cap = g.edges()
    part = (cap * rng.random(cap.shape[0])).astype(np.int32)
    z = rng.integers(0, g.n, size=(200, 2))
    loops = rng.integers(0, g.n, size=50)
    src2 = np.concatenate([src, src, z[:, 0], loops])
    dst2 = np.concatenate([dst, dst, z[:, 1], loops])
    cap2 = np.concatenate([part, cap - part, np.zeros(200, np.int32), rng.integers(1, 9, 50).astype(np.int32)])
    h = synth.shuffle_rows(synth.from_edges(g.n, src2, dst2, cap2, g.s, g.t), seed)
    q = oracle.maxflow_graph(h)
    assert q.flow == r.flow
    assert np.array_equal(q.in_S, r.in_S)
    check.check_flow(h.n, h.row_off, h.col, h.cap, h.s, h.t, q.flow, q.in_S, q.edge_flow, strict=True)


def test_bitmap_packing():
    r = oracle.OracleResult(0, 0, np.array([1, 0, 1] + [0] * 30 + [1], np.uint8), None, {}, 0.0)
    w = r.bitmap_words()
    assert w.dtype == np.uint32 and list(w) == [0b101, 0b10]


# ------------------------------------------------------------------ DIMACS-shaped generators (NEXT #4)
def test_dimacs_shapes_sizes():
    # structure decoded from Table 1: Washington-RLG 512x512x3 and Genrmf a=b=128
    g = synth.washington_rlg()
    assert (g.n, g.m) == (262146, 785920)
    L = synth._L()
    assert (128 * 128 * 128, L.synth_genrmf_count(128, 128)) == (2097152, 10403840)


@pytest.mark.parametrize("maker", [lambda: synth.washington_rlg(40, 50, 3, 100, 2), lambda: synth.genrmf(8, 10, 1, 100, 3)])
def test_dimacs_shapes_vs_scipy(maker):
    g = maker()
    r = oracle.maxflow_graph(g)
    assert r.flow == _scipy_flow(g) == r.cut_capacity
    check.check_flow(g.n, g.row_off, g.col, g.cap, g.s, g.t, r.flow, r.in_S, r.edge_flow, strict=True)
