"""-m gpu: dataset files run end to end through the C-ABI (NEXT #4).  A DIMACS
file (Genrmf / Washington-RLG shapes written by synth and read back by the DIMACS reader), a
SNAP edge list with the paper's 20-pair super terminals and a KONECT bipartite
list are solved on the GPU and compared bit-exactly with the oracle (F, cut
capacity, canonical bitmap; matching size = oracle F and a valid matching)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import matching
from tests.gpu_helpers import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("layout", ["bcsr", "rcsr"])
@pytest.mark.parametrize("make", [lambda: synth.genrmf(12, 10, seed=4),
                                  lambda: synth.washington_rlg(64, 64, 3, seed=2)], ids=["genrmf", "rlg"])
def test_dimacs_file_end_to_end(tmp_path, make, layout):
    p = str(tmp_path / "g.max")
    synth.write_dimacs(make(), p)
    assert_parity(synth.read_dimacs(p), layout)


def test_snap_file_end_to_end(tmp_path):
    src, dst, _ = synth.rmat_edges(12, 8, seed=9)
    ids = np.random.default_rng(1).choice(10**8, size=1 << 12, replace=False)
    p = tmp_path / "snap.txt"
    with open(p, "w") as f:
        f.write("# FromNodeId\tToNodeId\n")
        f.writelines(f"{a}\t{b}\n" for a, b in zip(ids[src], ids[dst]))
    g = synth.snap_instance(str(p), npairs=20, nstarts=256, seed=1)
    for layout in ("bcsr", "rcsr"):
        assert_parity(g, layout)


def test_konect_file_end_to_end(tmp_path):
    import torch
    import paper_2404_00270_b200 as W
    l, r = synth.bipartite_edges(3000, 2000, 9000, 5)
    p = tmp_path / "out.konect"
    with open(p, "w") as f:
        f.write(f"% bip unweighted\n% {l.size} 3000 2000\n")
        f.writelines(f"{a + 1} {b + 1} 1\n" for a, b in zip(l, r))
    nL, nR, l2, r2 = synth.read_konect(str(p))
    assert (nL, nR, l2.size) == (3000, 2000, l.size)
    size, match, _ = W.bipartite_match(nL, nR, torch.from_numpy(l2).cuda(), torch.from_numpy(r2).cuda())
    n, s, d, c, S, T = matching.network(nL, nR, l2, r2)
    assert size == oracle.maxflow_graph(synth.from_edges(n, s, d, c, S, T), phase2=False).flow
    matching.check_matching(nL, nR, l2, r2, match.cpu().numpy(), size)
