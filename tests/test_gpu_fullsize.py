"""-m gpu parity at the BENCHMARKED sizes (BASELINE.json configs C2-C5, the exact instances
bench.py times): flow value, cut capacity and canonical cut bitmap bit-exact against the
oracle on every instance (north_star: "exact max-flow values and min-cut capacities on every
generated instance"; SURVEY §4 tier 5 corpus).  The oracle runs on a thread pool over the
host cores (its C solver has no global state; ctypes releases the GIL per call).

Marked `slow` as well: about two minutes, most of it instance generation and the oracle."""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import matching
from tests.gpu_helpers import bits_to_mask, gpu_solve, to_dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_CACHE = {}


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_00270_b200 as W
    W.load()


def _oracle_many(graphs):
    oracle.build()
    with cf.ThreadPoolExecutor(max(1, _cores())) as ex:
        return list(ex.map(lambda g: oracle.maxflow_graph(g, phase2=False), graphs))


def _graph(name):
    if name not in _CACHE:
        if name in ("c3", "c3h"):
            _CACHE[name] = synth.rmat(22, 16, 1, "paper" if name == "c3" else "hub20")
        elif name == "c2":
            _CACHE[name] = synth.grid(1024, 1024, False, 1)
        elif name == "c2r":
            _CACHE[name] = synth.grid(1024, 1024, True, 1)
    return _CACHE[name]


def _oracle_of(name):
    key = ("oracle", name)
    if key not in _CACHE:
        _CACHE[key] = _oracle_many([_graph(name)])[0]
    return _CACHE[key]


def test_c5_all_64_instances_bitexact():
    """C5 exactly as bench.py solves it: the 64 R-MAT-18 instances (seeds 1000-1063, paper-rule
    terminals) as ONE disjoint-union batch; every instance's F, cut capacity and bitmap slice
    compared with the oracle."""
    import paper_2404_00270_b200 as W
    parts = synth.c5_batch(64)
    B = synth.disjoint_union(parts)
    ro, col, cap = to_dev(B.union)
    flows, cuts, bm, st = W.maxflow_batch(ro, col, cap, B.vbase, B.s, B.t, gr_gamma=0.5)
    mask = bits_to_mask(bm.cpu().numpy().view(np.uint32), B.union.n)
    refs = _oracle_many(parts)
    bad = []
    for i, (g, ref) in enumerate(zip(parts, refs)):
        if not (flows[i] == ref.flow and cuts[i] == ref.cut_capacity and
                np.array_equal(mask[B.vbase[i]:B.vbase[i + 1]], ref.in_S)):
            bad.append(i)
    assert not bad, f"instances differing from the oracle: {bad}"
    assert st["flow_value"] == sum(r.flow for r in refs)


@pytest.mark.parametrize("name,layout", [("c3", "bcsr"), ("c3", "rcsr"), ("c3h", "bcsr"), ("c3h", "rcsr"),
                                         ("c2", "bcsr"), ("c2", "rcsr"), ("c2r", "bcsr")])
def test_single_graph_configs_bitexact(name, layout):
    """C3 (R-MAT-22: paper-rule and hub20 terminals) and C2 (1024^2 grid: unit and U[1,100]
    capacities) at full size, both layouts where the bench quotes them."""
    g = _graph(name)
    F, words, st, _ = gpu_solve(g, layout)
    ref = _oracle_of(name)
    assert F == ref.flow and st["cut_capacity"] == ref.cut_capacity
    assert np.array_equal(words, ref.bitmap_words())
    if name == "c2":
        assert F == 1024      # closed form: 1024 disjoint unit row paths


@pytest.mark.parametrize("layout", ["bcsr", "rcsr"])
def test_c4_matching_full_size(layout):
    """C4: 2^20 x 2^20, 2^24 draws: matching size == the oracle's max-flow value on the same
    network, and the matching is valid (pairs are input edges, each vertex at most once)."""
    import torch
    import paper_2404_00270_b200 as W
    if "c4" not in _CACHE:
        l, r = synth.bipartite_edges(1 << 20, 1 << 20, 1 << 24, 1)
        n, src, dst, cap, s, t = matching.network(1 << 20, 1 << 20, l, r)
        _CACHE["c4"] = (l, r, _oracle_many([synth.from_edges(n, src, dst, cap, s, t)])[0].flow)
    l, r, F = _CACHE["c4"]
    size, match, st = W.bipartite_match(1 << 20, 1 << 20, torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda(),
                                        layout=layout)
    assert size == F == st["cut_capacity"]
    matching.check_matching(1 << 20, 1 << 20, l, r, match.cpu().numpy(), size)
