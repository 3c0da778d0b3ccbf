"""-m gpu tests of INTERMEDIATE device state (SURVEY.md §4 tier 3, §8(c) "Intermediate GPU
state"): the labels of a global relabel equal a host BFS over the same
residual graph, the compacted active-vertex queue equals the sequential predicate, and the
state right after the preflow + first GR equals the oracle's `initial_state` exactly.

The solve is stopped with the `debug_stop` option right after the compaction that follows
the k-th global relabel (wbpr.h); the residual view then exposes h, e, cf and the AVQ.
Also: EOVERFLOW on antiparallel pairs whose capacities sum past INT32_MAX, the bottom-up /
top-down split of the BFS counters, and the per-warp trace summing to the solve counters."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import oracle
import synth
from oracle import check
from tests.gpu_helpers import dense_bcsr, gpu_solve, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_00270_b200 as W
    W.load()


def _stopped(g, k, **opt):
    """Solve with debug_stop=k; returns (residual view dict, dense BCSR, stats)."""
    import paper_2404_00270_b200 as W
    F, words, st, ws = gpu_solve(g, "bcsr", debug_stop=k, **opt)
    R = W.residual(ws)
    return R, dense_bcsr(R), st


def _host_levels(n, D, t):
    """Reverse BFS distance to t over the residual arcs u -> col with cf > 0,
    computed on the host from the device's own residual state; unreachable = -1."""
    owner = np.repeat(np.arange(n), np.diff(D["off"].astype(np.int64)))
    live = D["cf"] > 0
    # reversed arcs col -> u, so a BFS from t follows residual arcs backwards
    A = sp.csr_matrix((np.ones(int(live.sum())), (D["col"][live], owner[live])), shape=(n, n))
    d = shortest_path(A, method="D", unweighted=True, indices=int(t))
    return np.where(np.isinf(d), -1, d).astype(np.int64)


def _check_labels_and_avq(g, R, D):
    n, s, t = g.n, g.s, g.t
    h, e = R["h"].astype(np.int64), R["e"]
    lv = _host_levels(n, D, t)
    others = np.ones(n, bool)
    others[[s, t]] = False
    want = np.where(lv >= 0, lv, n)
    assert h[t] == 0 and h[s] == n + 1          # sinks 0, sources n + 1 (DESIGN reading #7)
    bad = np.nonzero((h != want) & others)[0]
    assert bad.size == 0, f"GR labels differ from the host BFS at {bad[:10]} ({h[bad[:10]]} vs {want[bad[:10]]})"
    # AVQ = {v not in {s,t}: e(v) > 0 and h(v) < n} (Alg. 2 l.1-4), each once
    avq = np.sort(R["avq"])
    assert np.unique(avq).size == avq.size, "a vertex was queued twice"
    pred = np.nonzero(others & (e > 0) & (h < n))[0]
    assert np.array_equal(avq, pred), "AVQ differs from the sequential predicate"
    # invariants at the barrier: cf >= 0, pair conservation, e = net inflow >= 0
    f = check.demerge_bcsr(n, g.row_off, g.col, g.cap, D["off"], D["col"], D["cf"], D["cap0"], D["mate"])
    src = np.repeat(np.arange(n), np.diff(g.row_off))
    net = (np.bincount(g.col, weights=f, minlength=n) - np.bincount(src, weights=f, minlength=n)).astype(np.int64)
    assert np.array_equal(net[others], e[others]), "excess differs from the net inflow of the residual state"
    assert np.all(e[others] >= 0)
    # Excess_total after the compaction: initial total minus the excess frozen on
    # vertices that cannot reach t
    return h, e


GRAPHS = [
    lambda: synth.tiny_random(9, 30, 5, 3),
    lambda: synth.tiny_random(12, 60, 8, 11),
    lambda: synth.random_graph(1024, 8192, 2),
    lambda: synth.grid(24, 18, True, 3),
    lambda: synth.rmat(11, 16, 5, "hub20"),
    lambda: synth.rmat(12, 16, 4, "paper"),
]


@pytest.mark.parametrize("gi", range(len(GRAPHS)))
def test_first_gr_equals_oracle_initial_state(gi):
    """debug_stop=1: preflow (Alg. 1 Step 0) + one exact GR are
    deterministic, so e, h and Excess_total equal oracle.initial_state bit-exactly."""
    g = GRAPHS[gi]()
    R, D, st = _stopped(g, 1)
    e0, tot, lv, _ = oracle.initial_state(g.n, g.row_off, g.col, g.cap, g.s, g.t)
    h, e = _check_labels_and_avq(g, R, D)
    others = np.ones(g.n, bool)
    others[[g.s, g.t]] = False
    assert np.array_equal(e[others], e0[others]) and e[g.t] == e0[g.t]
    assert np.array_equal(h[others], lv[others])          # oracle: unreached = n as well
    frozen = others & (lv >= g.n)
    assert R["excess_total"] == tot - int(e0[frozen].sum())
    assert st["global_relabels"] == 1 and st["rounds"] == 0


@pytest.mark.parametrize("gi", range(len(GRAPHS)))
@pytest.mark.parametrize("k", [2, 3, 5])
def test_later_gr_labels_and_avq(gi, k):
    """debug_stop=k after rounds of push/relabel (a nondeterministic trajectory): the labels
    of the k-th GR equal a host BFS over the device's own residual graph and the AVQ equals
    the sequential predicate.  gr_beta small forces frequent GRs."""
    g = GRAPHS[gi]()
    for bfs_mode in (0, 1, 2):
        R, D, st = _stopped(g, k, gr_beta=0.02, bfs_mode=bfs_mode, small_mode=0)
        assert st["global_relabels"] <= k
        _check_labels_and_avq(g, R, D)


def test_small_mode_gr_labels():
    """Same check with the small-frontier CTA mode on (GRs triggered from CTA 0)."""
    g = synth.grid(40, 30, True, 2)
    for k in (2, 4):
        R, D, _ = _stopped(g, k, small_mode=1)
        _check_labels_and_avq(g, R, D)


def test_debug_stop_rejects_batches_and_phase2():
    import paper_2404_00270_b200 as W
    g = synth.tiny_random(9, 30, 5, 3)
    with pytest.raises(W.WbprError) as e:
        gpu_solve(g, "bcsr", debug_stop=1, phase2=1)
    assert e.value.name == "WBPR_EINVAL"


# ------------------------------------------------------------------ EOVERFLOW on antiparallel pairs
@pytest.mark.parametrize("c", [2**31 - 1, 2**30 + 1])
def test_antiparallel_pair_overflow(c):
    """BCSR stores u->v and v->u as ONE arc pair whose residual capacities always sum to
    c(u,v) + c(v,u) (a push moves d between them); past INT32_MAX the int32 cf would wrap,
    so the build reports EOVERFLOW.  RCSR keeps the two arcs distinct and solves it."""
    import paper_2404_00270_b200 as W
    g = synth.from_edges(3, [0, 1, 1], [1, 0, 2], [c, c, 5], 0, 2)
    with pytest.raises(W.WbprError) as e:
        gpu_solve(g, "bcsr")
    assert e.value.name == "WBPR_EOVERFLOW"
    F, _, _, _ = gpu_solve(g, "rcsr")
    assert F == 5


def test_antiparallel_pair_at_limit_ok():
    """c(u,v) + c(v,u) = INT32_MAX exactly is representable: solved normally."""
    c1 = 2**30
    g = synth.from_edges(3, [0, 1, 1], [1, 0, 2], [c1, 2**31 - 1 - c1, 7], 0, 2)
    F, _, st, _ = gpu_solve(g, "bcsr")
    assert F == 7 == st["cut_capacity"]


# ------------------------------------------------------------------ counters
def test_bfs_counter_split():
    """bfs_arcs_bottom_up is the bottom-up part of bfs_arcs_scanned: 0 with top-down only,
    every BFS arc with bottom-up from level 1 (bfs_mode 2 still scans level 0 top-down)."""
    g = synth.rmat(14, 16, 2, "hub20")
    ref = oracle.maxflow_graph(g, phase2=False)
    F0, _, s0, _ = gpu_solve(g, "bcsr", bfs_mode=0)
    F1, _, s1, _ = gpu_solve(g, "bcsr", bfs_mode=1)
    F2, _, s2, _ = gpu_solve(g, "bcsr", bfs_mode=2)
    assert F0 == F1 == F2 == ref.flow
    assert s0["bfs_arcs_bottom_up"] == 0 < s0["bfs_arcs_scanned"]
    assert 0 <= s1["bfs_arcs_bottom_up"] <= s1["bfs_arcs_scanned"]
    assert 0 < s2["bfs_arcs_bottom_up"] <= s2["bfs_arcs_scanned"]


@pytest.mark.parametrize("schedule", ["vc", "tc"])
def test_trace_sums_to_counters(schedule):
    """With every grid round traced (small mode off), the per-warp records sum to the solve's
    own counters: slots scanned, pushes and relabels (NEXT #3 bookkeeping)."""
    import paper_2404_00270_b200 as W
    g = synth.rmat(12, 16, 3, "hub20")
    ro, col, cap = to_dev(g)
    opt = W.options("bcsr", schedule=schedule, trace_rounds=256, small_mode=0)
    ws = W.Workspace(W.workspace_size(g.n, g.m, 1, opt))
    F, _, st = W.maxflow(ro, col, cap, g.s, g.t, workspace=ws, schedule=schedule, trace_rounds=256, small_mode=0)
    assert st["rounds"] <= 256
    rec = W.trace(ws)
    assert int(rec["slots"].sum()) == st["arcs_scanned"]
    assert int(rec["pushes"].sum()) == st["pushes"]
    assert int(rec["relabels"].sum()) == st["relabels"]
