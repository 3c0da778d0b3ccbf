"""-m gpu: the one-CTA fused path for tiny single instances (tiny.cu, option tiny_mode).

Both paths must give the oracle's unique results (F, cut capacity, canonical bitmap; §8(c) N6)
and a residual state that passes V1-V7, on the same inputs: adversarial tiny graphs (parallel,
antiparallel, zero-capacity edges, self-loops), C1 seeds, small grids and R-MATs, a hub, the
size limits of the path, and the error returns."""
import numpy as np
import pytest

import oracle
import synth
from oracle import brute
from tests.gpu_helpers import assert_parity, gpu_solve, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_path_selection():
    g = synth.random_graph(1024, 8192, 1)
    _, _, st, _ = gpu_solve(g)
    assert st["tiny_path"] == 1 and st["kernel_launches"] == 1
    _, _, st, _ = gpu_solve(g, tiny_mode=1)
    assert st["tiny_path"] == 0 and st["kernel_launches"] > 1
    for opt in (dict(layout="rcsr"), dict(push_mode=0), dict(schedule="tc"), dict(phase2=1), dict(gap_mode=1),
                dict(grid_blocks=2)):
        layout = opt.pop("layout", "bcsr")
        _, _, st, _ = gpu_solve(g, layout, **opt)
        assert st["tiny_path"] == 0, opt


@pytest.mark.parametrize("tiny_mode", [0, 1])
def test_tiny_random_brute_force(tiny_mode):
    for seed in range(120):
        rng = np.random.default_rng(70_000 + seed)
        n = int(rng.integers(2, 12))
        g = synth.tiny_random(n, int(rng.integers(0, 40)), int(rng.integers(1, 9)), seed)
        F, st = assert_parity(g, tiny_mode=tiny_mode)
        assert st["tiny_path"] == (1 - tiny_mode)
        if n <= 10:
            c, _ = brute.enum_mincut(g.n, g.row_off, g.col, g.cap, g.s, g.t)
            assert F == c


@pytest.mark.parametrize("seed", range(1, 9))
def test_c1_both_paths(seed):
    g = synth.random_graph(1024, 8192, seed)
    ref = oracle.maxflow_graph(g, phase2=False)
    F0, st0 = assert_parity(g, ref=ref)
    F1, st1 = assert_parity(g, ref=ref, tiny_mode=1)
    assert st0["tiny_path"] == 1 and st1["tiny_path"] == 0 and F0 == F1 == ref.flow


@pytest.mark.parametrize("make", [lambda: synth.grid(40, 40, True, 2), lambda: synth.grid(30, 30, False),
                                  lambda: synth.rmat(10, 7, 3, "paper"), lambda: synth.rmat(10, 7, 4, "hub20"),
                                  lambda: synth.washington_rlg(20, 30, 3, 100, 2)],
                         ids=["grid-rand", "grid-unit", "rmat-paper", "rmat-hub", "rlg"])
def test_shapes(make):
    g = make()
    assert 2 * g.m <= 16384 and g.n <= 2048
    _, st = assert_parity(g)
    assert st["tiny_path"] == 1


def test_hub_and_limits():
    # a hub with > 1024 slots; n = 2048 and 2m = 16384 exactly (the path's limits), then one
    # edge more (the multi-kernel path)
    rng = np.random.default_rng(5)
    n = 2048
    src = np.concatenate([np.zeros(1500, np.int64), rng.integers(0, n, 8192 - 1500)])
    dst = np.concatenate([rng.choice(np.arange(1, n), 1500, replace=False), rng.integers(0, n, 8192 - 1500)])
    cap = rng.integers(0, 50, 8192)
    g = synth.from_edges(n, src, dst, cap, 0, n - 1)
    _, st = assert_parity(g)
    assert st["tiny_path"] == 1
    g2 = synth.from_edges(n, np.append(src, 3), np.append(dst, 4), np.append(cap, 7), 0, n - 1)
    _, st = assert_parity(g2)
    assert st["tiny_path"] == 0


@pytest.mark.parametrize("tiny_mode", [0, 1])
def test_errors_both_paths(tiny_mode):
    import paper_2404_00270_b200 as W
    g = synth.random_graph(100, 400, 1, 0, 99)
    ro, col, cap = to_dev(g)
    bad = col.clone(); bad[17] = 100
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro, bad, cap, 0, 99, tiny_mode=tiny_mode)
    assert e.value.name == "WBPR_EINVAL"
    neg = cap.clone(); neg[3] = -1
    with pytest.raises(W.WbprError) as e:
        W.maxflow(ro, col, neg, 0, 99, tiny_mode=tiny_mode)
    assert e.value.name == "WBPR_EINVAL"
    badro = ro.clone(); badro[5] = badro[6] + 1
    with pytest.raises(W.WbprError) as e:
        W.maxflow(badro, col, cap, 0, 99, tiny_mode=tiny_mode)
    assert e.value.name == "WBPR_EINVAL"
    # parallel edges summing past INT32_MAX, and an antiparallel pair whose two residual
    # capacities would
    for srcs, dsts, caps in (([0, 0, 0, 1], [1, 1, 1, 2], [2**30] * 3 + [5]),
                             ([0, 1, 1], [1, 0, 2], [2**31 - 1, 2**31 - 1, 5])):
        h = synth.from_edges(3, srcs, dsts, caps, 0, 2)
        r2, c2, k2 = to_dev(h)
        with pytest.raises(W.WbprError) as e:
            W.maxflow(r2, c2, k2, 0, 2, tiny_mode=tiny_mode)
        assert e.value.name == "WBPR_EOVERFLOW"


def test_host_buffers():
    # the C-ABI's host-buffer form (copies inside the call) on the tiny path
    import torch
    import paper_2404_00270_b200 as W
    g = synth.random_graph(1024, 8192, 3)
    ro, col, cap = (torch.from_numpy(a) for a in (g.row_off, g.col, g.cap))
    F, bm, st = W.maxflow(ro, col, cap, g.s, g.t)
    ref = oracle.maxflow_graph(g, phase2=False)
    assert st["tiny_path"] == 1 and F == ref.flow
    assert np.array_equal(bm.numpy().view(np.uint32), ref.bitmap_words())
