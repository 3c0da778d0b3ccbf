"""-m gpu parity tests: the CUDA path (through the C-ABI) against the oracle on
the same seeded inputs.  Integer results must match bit-exactly: flow value,
min-cut capacity and the canonical cut bitmap (unique); the
flow assignment (not unique) must pass V1-V7."""
import numpy as np
import pytest

import oracle
import synth
from oracle import brute, matching, residual_ref
from tests.gpu_helpers import assert_parity, bits_to_mask, dense_bcsr, gpu_solve, to_dev

pytestmark = pytest.mark.gpu
LAYOUTS = ["bcsr", "rcsr"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_00270_b200 as W
    W.load()


# ------------------------------------------------------------------ A1 construction, bit-exact
def _build(g, layout):
    import paper_2404_00270_b200 as W
    ro, col, cap = to_dev(g)
    return W.build_residual(ro, col, cap, layout=layout)


BUILD_CASES = [("tiny", s) for s in range(12)] + [("c1", 1), ("grid", 1), ("rmat", 3), ("hubs", 0),
                                                  ("sorted_rmat", 4), ("bip", 1)] + [("runs", s) for s in range(3)]


def _runs_graph(seed):
    """Segments sized around the merge-class boundaries (thread class <= 12 elements, warp
    windows of 32 outputs, 64, 96) with runs of parallel and antiparallel half-arcs placed
    across the 32-output window boundaries: the warp merge's register run sums and their
    global continuation, and the next-window prefetch (merge.cu)."""
    rng = np.random.default_rng(100 + seed)
    n = 600
    src, dst = [], []
    for p_, size in enumerate([11, 12, 13, 14, 20, 31, 32, 33, 34, 40, 63, 64, 65, 96, 97, 130]):
        u = p_
        d_in = size // 3
        cols = list(rng.choice(np.arange(200, n), size=size - d_in, replace=False))
        # parallel copies of the columns that land around output positions 28-36 and 60-68
        sc = sorted(cols)
        for k in (27, 29, 30, 31, 32, 33, 62, 63, 64):
            if k < len(sc):
                cols += [sc[k]] * int(rng.integers(1, 3))
        for c in cols:
            src.append(u); dst.append(c)
        # in-arcs: some antiparallel (from columns u points to), some from elsewhere
        ins = list(rng.choice(sc, size=min(d_in // 2, len(sc)), replace=False)) + \
            list(rng.integers(20, n, size=d_in - d_in // 2))
        for v in ins:
            src.append(int(v)); dst.append(u)
            if rng.random() < 0.3:
                src.append(int(v)); dst.append(u)    # parallel in-edge
    # background edges so that s and t connect through the probe vertices
    for _ in range(3000):
        a, b = rng.integers(0, n, 2)
        if a != b:
            src.append(int(a)); dst.append(int(b))
    src, dst = np.array(src, np.int64), np.array(dst, np.int64)
    cap = rng.integers(0, 60, src.shape[0]).astype(np.int32)
    return synth.shuffle_rows(synth.from_edges(n, src, dst, cap, 0, n - 1, name=f"runs{seed}"), seed)


def _build_graph(kind, seed):
    if kind == "tiny":
        return synth.tiny_random(12 + seed, 60 + 10 * seed, 6, seed)
    if kind == "c1":
        return synth.shuffle_rows(synth.random_graph(1024, 8192, seed), seed)
    if kind == "grid":
        return synth.grid(37, 23, True, seed)
    if kind == "rmat":
        return synth.shuffle_rows(synth.rmat(13, 16, seed, "hub20"), seed)
    if kind == "hubs":
        # segments of every size class: <=32, <=4096, > 4096 (merge passes), duplicates
        rng = np.random.default_rng(7)
        n = 20000
        # vertex 2: > 8192 in-arcs (chunked merge), some parallel; vertex 0: 9000 unsorted out-arcs
        src = np.concatenate([np.zeros(9000, np.int64), np.full(5000, 1), rng.integers(0, n, 30000), [5, 5, 5],
                              rng.integers(3, n, 12000)])
        dst = np.concatenate([rng.integers(0, n, 9000), rng.integers(0, n, 5000), rng.integers(0, n, 30000), [5, 6, 6],
                              np.full(12000, 2)])
        cap = rng.integers(0, 50, src.shape[0]).astype(np.int32)
        return synth.shuffle_rows(synth.from_edges(n, src, dst, cap, 0, n - 1), 3)
    if kind == "runs":
        return _runs_graph(seed)
    if kind == "sorted_rmat":   # rows already column-sorted (no out-row sort needed)
        return synth.rmat(12, 16, seed, "paper")
    if kind == "bip":           # 2^12 x 2^12 matching network: s and t are hubs
        l, r = synth.bipartite_edges(1 << 13, 1 << 13, 1 << 15, seed)
        n, src, dst, cap, s, t = matching.network(1 << 13, 1 << 13, l, r)
        return synth.shuffle_rows(synth.from_edges(n, src, dst, cap, s, t), seed)
    raise ValueError(kind)


@pytest.mark.parametrize("kind,seed", BUILD_CASES)
def test_build_bcsr_bitexact(kind, seed):
    g = _build_graph(kind, seed)
    G, st = _build(g, "bcsr")
    R = dense_bcsr(G)
    ref = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
    assert R["M"] == ref["col"].shape[0] == st["M"]
    assert np.array_equal(R["off"], ref["off"])
    assert np.array_equal(R["col"], ref["col"])
    assert np.array_equal(R["cf"], ref["cf0"])
    assert np.array_equal(R["cap0"], ref["cf0"])
    assert np.array_equal(R["mate"], ref["mate"])
    src, dst, _ = g.edges()
    assert st["self_loops_ignored"] == int((src == dst).sum())


@pytest.mark.parametrize("kind,seed", BUILD_CASES)
def test_build_rcsr_bitexact(kind, seed):
    g = _build_graph(kind, seed)
    R, _ = _build(g, "rcsr")
    ref = residual_ref.rcsr(g.n, g.row_off, g.col, g.cap)
    assert np.array_equal(R["foff"], ref["foff"])
    assert np.array_equal(R["fcol"], ref["fcol"])
    assert np.array_equal(R["fcf"], ref["fcf0"])
    assert np.array_equal(R["roff"], ref["roff"])
    assert np.array_equal(R["rcol"], ref["rcol"])
    assert np.array_equal(R["fidx"], ref["fidx"])
    assert np.all(R["bcf"] == 0)


# ------------------------------------------------------------------ end-to-end parity
@pytest.mark.parametrize("layout", LAYOUTS)
def test_spec_examples(golden, layout):
    for ex in golden["maxflow"]:
        e = np.array(ex["edges"], np.int64).reshape(-1, 3)
        g = synth.from_edges(ex["n"], e[:, 0], e[:, 1], e[:, 2], ex["s"], ex["t"])
        F, _ = assert_parity(g, layout)
        assert F == ex["flow"], ex["citation"]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("chunk", range(4))
def test_tiny_random_vs_brute_force(layout, chunk):
    for seed in range(chunk * 60, chunk * 60 + 60):
        rng = np.random.default_rng(50_000 + seed)
        n = int(rng.integers(2, 12))
        g = synth.tiny_random(n, int(rng.integers(0, 40)), int(rng.integers(1, 9)), seed)
        F, _ = assert_parity(g, layout)
        if n <= 10:
            c, S_max = brute.enum_mincut(g.n, g.row_off, g.col, g.cap, g.s, g.t)
            assert F == c


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("seed", range(1, 17))
def test_c1_seeds(layout, seed):
    assert_parity(synth.random_graph(1024, 8192, seed), layout)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_random_grid(layout):
    assert_parity(synth.grid(64, 48, True, 5), layout)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("k", [16, 128])
def test_unit_grid_closed_form(layout, k):
    F, _ = assert_parity(synth.grid(k, k, False), layout)
    assert F == k


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("rule", ["paper", "hub20"])
def test_rmat14(layout, rule):
    assert_parity(synth.rmat(14, 16, 2, rule), layout)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_huge_vertex_chunks(layout):
    # a hub with > kChunk slots that must discharge through many rounds
    rng = np.random.default_rng(11)
    n = 6000
    hub = 1
    src = np.concatenate([[0], np.full(5000, hub), rng.integers(2, n - 1, 20000)])
    dst = np.concatenate([[hub], rng.integers(2, n - 1, 5000), rng.integers(2, n, 20000)])
    cap = np.concatenate([[10**6], rng.integers(1, 20, 25000)]).astype(np.int32)
    g = synth.from_edges(n, src, dst, cap, 0, n - 1)
    assert_parity(g, layout)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_gr_frequency_and_grid_size_invariance(layout):
    g = synth.random_graph(3000, 24000, 9, 0, 2999)
    ref = oracle.maxflow_graph(g, phase2=False)
    for beta, blocks in ((0.02, 0), (5.0, 0), (0.5, 3), (0.5, 1)):
        assert_parity(g, layout, ref=ref, validate=False, gr_beta=beta, grid_blocks=blocks)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("push_mode", [0, 1])
@pytest.mark.parametrize("bfs_mode", [0, 1, 2, 3])
@pytest.mark.parametrize("small_mode", [0, 1])
@pytest.mark.parametrize("gap_mode", [0, 1])
def test_modes(layout, push_mode, bfs_mode, small_mode, gap_mode):
    # the paper's single push (Alg. 2) and the discharge deviation; top-down, direction-
    # optimizing and bottom-up BFS: all must reach the same unique F / cut / S*
    for g in (synth.rmat(12, 16, 7, "hub20"), synth.grid(40, 30, True, 2),
              synth.tiny_random(9, 30, 5, 3), synth.random_graph(800, 6000, 5, 0, 799)):
        assert_parity(g, layout, push_mode=push_mode, bfs_mode=bfs_mode, small_mode=small_mode, gap_mode=gap_mode)


# ------------------------------------------------------------------ host-buffer path (e2e)
def test_host_buffers():
    import torch
    import paper_2404_00270_b200 as W
    g = synth.random_graph(1024, 8192, 3)
    ref = oracle.maxflow_graph(g, phase2=False)
    ro, col, cap = (torch.from_numpy(a).pin_memory() for a in (g.row_off, g.col, g.cap))
    F, bm, st = W.maxflow(ro, col, cap, g.s, g.t)
    assert not bm.is_cuda
    assert F == ref.flow and np.array_equal(bm.numpy().view(np.uint32), ref.bitmap_words())


# ------------------------------------------------------------------ bipartite (A9)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("seed", range(4))
def test_bipartite(layout, seed):
    import torch
    import paper_2404_00270_b200 as W
    nL, nR = 3000 + 100 * seed, 2500
    l, r = synth.bipartite_edges(nL, nR, 7000, seed)
    n, src, dst, cap, s, t = matching.network(nL, nR, l, r)
    ref = oracle.maxflow_graph(synth.from_edges(n, src, dst, cap, s, t), phase2=False).flow
    size, match, st = W.bipartite_match(nL, nR, torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda(), layout=layout)
    assert size == ref
    matching.check_matching(nL, nR, l, r, match.cpu().numpy(), size)


def test_bipartite_spec_examples(golden):
    import torch
    import paper_2404_00270_b200 as W
    for ex in golden["matching"]:
        l = torch.tensor([e[0] for e in ex["edges"]], dtype=torch.int32, device="cuda")
        r = torch.tensor([e[1] for e in ex["edges"]], dtype=torch.int32, device="cuda")
        size, match, _ = W.bipartite_match(ex["nL"], ex["nR"], l, r)
        assert size == ex["size"], ex["citation"]


# ------------------------------------------------------------------ batch (A10)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("groups", [0, 2, 5, 11])
@pytest.mark.parametrize("phase2", [0, 1])
def test_batch_union(layout, groups, phase2):
    # groups 0 / 1: one solver for the union (default); 2 / 5: contiguous instance ranges per
    # solver group
    import torch
    import paper_2404_00270_b200 as W
    parts = [synth.rmat(11, 16, 100 + i, "paper" if i % 2 else "hub20") for i in range(6)]
    parts += [synth.random_graph(500, 3000, i, 0, 499) for i in range(3)]
    parts += [synth.grid(20, 15, True, 4), synth.tiny_random(8, 20, 5, 2, self_loops=False, s=0, t=7)]
    B = synth.disjoint_union(parts)
    ro, col, cap = to_dev(B.union)
    flows, cuts, bm, st = W.maxflow_batch(ro, col, cap, B.vbase, B.s, B.t, layout=layout, batch_groups=groups,
                                          phase2=phase2)
    mask = bits_to_mask(bm.cpu().numpy().view(np.uint32), B.union.n)
    for i, g in enumerate(parts):
        ref = oracle.maxflow_graph(g, phase2=False)
        assert flows[i] == ref.flow and cuts[i] == ref.flow
        assert np.array_equal(mask[B.vbase[i]:B.vbase[i + 1]], ref.in_S)


# ------------------------------------------------------------------ errors
def test_errors():
    import torch
    import paper_2404_00270_b200 as W
    g = synth.random_graph(100, 400, 1, 0, 99)
    ro, col, cap = to_dev(g)
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro, col, cap, 5, 5)
    assert e.value.name == "WBPR_EINVAL"
    bad = col.clone(); bad[17] = 100
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro, bad, cap, 0, 99)
    assert e.value.name == "WBPR_EINVAL"
    neg = cap.clone(); neg[3] = -1
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro, col, neg, 0, 99)
    assert e.value.name == "WBPR_EINVAL"
    h = synth.from_edges(3, [0, 0, 0, 1], [1, 1, 1, 2], [2**30, 2**30, 2**30, 5], 0, 2)
    ro2, col2, cap2 = to_dev(h)
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro2, col2, cap2, 0, 2)
    assert e.value.name == "WBPR_EOVERFLOW"
    import ctypes
    L = W.load()
    c = W.wbpr._as_csr(ro, col, cap)
    small = W.Workspace(1024)
    rc = L.wbpr_maxflow_solve(ctypes.byref(c), 0, 99, ctypes.byref(W.options()), small.ptr, 1024, None, None,
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == -3  # WBPR_ENOMEM


# ------------------------------------------------------------------ thread-centric schedule (NEXT #1)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("push_mode", [0, 1])
def test_thread_centric(layout, push_mode):
    # Alg. 1 Step 1: one thread per vertex per sweep; same unique F / cut / S* as the VC path
    for g in (synth.rmat(12, 16, 7, "paper"), synth.rmat(11, 16, 3, "hub20"), synth.grid(30, 20, True, 1),
              synth.random_graph(600, 5000, 2, 0, 599), synth.tiny_random(10, 40, 6, 9)):
        assert_parity(g, layout, schedule="tc", push_mode=push_mode)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_dimacs_shapes(layout):
    for g in (synth.washington_rlg(64, 64, 3, 10000, 5), synth.genrmf(16, 16, 1, 10000, 5)):
        assert_parity(g, layout)


# ------------------------------------------------------------------ device phase 2 (NEXT #2)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("schedule", ["vc", "tc"])
def test_phase2_true_flow(layout, schedule):
    # after phase 2 the de-merged residual state is a true flow: V2 strict conservation
    gs = [synth.tiny_random(10, 40, 6, s) for s in range(20)]
    gs += [synth.random_graph(1024, 8192, 4), synth.rmat(12, 16, 5, "hub20"), synth.grid(40, 30, True, 3),
           synth.washington_rlg(30, 40, 3, 100, 1)]
    for g in gs:
        assert_parity(g, layout, phase2=1, schedule=schedule)


# ------------------------------------------------------------------ workload trace (NEXT #3)
def test_trace_vc_balances_better_than_tc():
    # SPEC acceptance 5 analogue: on a skewed graph the vertex-centric schedule's
    # mean-normalised per-warp busy-time spread is below the thread-centric one's
    import torch
    import paper_2404_00270_b200 as W
    g = synth.rmat(14, 16, 3, "hub20")
    ro, col, cap = to_dev(g)
    spread = {}
    for sch in ("tc", "vc"):
        opt = W.options("bcsr", schedule=sch, trace_rounds=8, small_mode=0)
        ws = W.Workspace(W.workspace_size(g.n, g.m, 1, opt))
        F, _, st = W.maxflow(ro, col, cap, g.s, g.t, workspace=ws, schedule=sch, trace_rounds=8, small_mode=0)
        rec = W.trace(ws)
        assert rec.shape[0] == 8 and rec.shape[1] == st["grid_blocks"] * st["block_threads"] // 32
        assert int(rec["pushes"].sum()) <= st["pushes"]
        vals = []
        for r in range(rec.shape[0]):
            act = rec[r][rec[r]["tasks"] > 0]
            if act.shape[0] > 1 and act["busy_ns"].mean() > 0:
                b = act["busy_ns"].astype(float)
                vals.append((b / b.mean()).std())
        spread[sch] = float(np.median(vals))
    assert spread["vc"] < spread["tc"], spread


@pytest.mark.parametrize("layout", LAYOUTS)
def test_phase_timing_consistency(layout):
    """wbpr_stats.phase_ns / phase_count: one GR reset and one compaction per global
    relabel, every grid-wide round counted, times positive and within the solve window."""
    g = synth.rmat(14, 16, 7, "hub20")
    F, words, st, _ = gpu_solve(g, layout)
    ref = oracle.maxflow_graph(g, phase2=False)
    assert F == ref.flow
    pc, pn = st["phase_count"], st["phase_ns"]
    assert pc[2] == st["global_relabels"] == pc[4]
    assert pc[5] == 1                                   # one preflow
    assert pc[1] <= st["rounds"]                        # (small-mode rounds are counted in pc[9])
    assert pc[3] + pc[8] <= st["bfs_levels"]
    assert all(x >= 0 for x in pn) and sum(pn) > 0
    assert sum(pn) <= st["solve_ms"] * 1e6 * 1.05


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("kind", ["grid", "rlg", "genrmf", "path"])
def test_async_gr_deep_graphs(layout, kind):
    """bfs_mode 3: GRs deeper than 32 levels continue as the asynchronous label-correcting
    BFS; F, cut capacity and the canonical bitmap must stay bit-exact and the residual state
    must pass V1-V7."""
    if kind == "grid":
        g = synth.grid(96, 64, True, 3)
    elif kind == "rlg":
        g = synth.washington_rlg(64, 32, 3, 1000, 2)
    elif kind == "genrmf":
        g = synth.genrmf(12, 10, 1, 1000, 4)
    else:
        k = 500
        src = np.arange(k - 1); dst = src + 1
        g = synth.from_edges(k, src, dst, np.full(k - 1, 3, np.int32), 0, k - 1)
    F, st = assert_parity(g, layout, bfs_mode=3)
    if kind != "path":
        assert st["phase_count"][7] > 0, "the asynchronous continuation did not run"


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("layout", LAYOUTS)
def test_runs_across_merge_windows_parity(seed, layout):
    """F, cut capacity and bitmap bit-exact on the merge-class boundary graphs (parallel and
    antiparallel runs across the warp-merge windows), and V1-V7 on the residual state."""
    assert_parity(_runs_graph(seed), layout)
