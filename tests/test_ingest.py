"""Dataset readers (NEXT #4; SPEC "ingest" module S:316-393; §4.1
P:427-434): DIMACS max-flow, SNAP edge lists, KONECT bipartite lists.  CPU only.

The SPEC worked examples are checked literally; the readers are round-tripped
through the DIMACS writer on generated DIMACS-shaped networks; the Table 1 / Table 2
sizes and matching values (tests/golden/paper_datasets.json, cited per row) are checked
when the dataset files are supplied through WBPR_DATASETS (they are not in the repo)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import matching

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _w(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


# ------------------------------------------------------------------ DIMACS
def test_dimacs_single_edge(tmp_path):
    # "p max 2 1 / n 1 s / n 2 t / a 1 2 5" -> 2 vertices, one cap-5 edge
    g = synth.read_dimacs(_w(tmp_path, "a.max", "p max 2 1\nn 1 s\nn 2 t\na 1 2 5\n"))
    assert (g.n, g.m, g.s, g.t) == (2, 1, 0, 1)
    assert g.col.tolist() == [1] and g.cap.tolist() == [5]
    assert oracle.maxflow_graph(g).flow == 5


def test_dimacs_crlf_comments_and_whitespace(tmp_path):
    txt = "c a comment\r\np  max 3 2 \r\nc another\r\nn 3 t\r\nn 1 s\r\na 1 2 4\r\na 2 3 7  \r\n"
    g = synth.read_dimacs(_w(tmp_path, "b.max", txt))
    assert (g.n, g.m, g.s, g.t) == (3, 2, 0, 2)
    assert oracle.maxflow_graph(g).flow == 4


@pytest.mark.parametrize("text,code,line", [
    ("c only comments\nc more\n", -2, 0),                      # MissingProblemLine
    ("p max 2 1\nn 1 s\na 1 2 5\n", -3, 0),                     # MissingSourceOrSink
    ("p max 2 1\nn 1 s\nn 2 t\na 1 2\n", -4, 4),                # MalformedLine with its number
    ("p max 2 1\nn 1 s\nn 2 t\na 1 3 5\n", -5, 4),              # id beyond N
    ("p max 2 1\nn 1 s\nn 2 t\na 1 2 -5\n", -6, 4),             # negative capacity
    ("p max 2 1\nn 1 s\nn 2 t\na 1 2 2147483648\n", -6, 4),     # capacity beyond int32
    ("a 1 2 5\np max 2 1\n", -2, 1),                            # arc before the problem line
    ("p max 2 1\nn 1 x\n", -4, 2),
])
def test_dimacs_errors(tmp_path, text, code, line):
    with pytest.raises(synth.IngestError) as ei:
        synth.read_dimacs(_w(tmp_path, "e.max", text))
    assert ei.value.code == code and ei.value.line == line


def test_dimacs_arc_count_mismatch_is_a_warning(tmp_path):
    g = synth.read_dimacs(_w(tmp_path, "c.max", "p max 2 3\nn 1 s\nn 2 t\na 1 2 5\n"))
    assert g.m == 1 and g.meta["declared_m"] == 3 and g.meta["arc_count_mismatch"]


def test_dimacs_missing_file():
    with pytest.raises(synth.IngestError) as ei:
        synth.read_dimacs("/nonexistent/x.max")
    assert ei.value.code == -1


@pytest.mark.parametrize("make", [
    lambda: synth.washington_rlg(16, 16, 3, seed=3),
    lambda: synth.genrmf(6, 5, seed=2),
    lambda: synth.tiny_random(9, 30, 5, seed=11),
])
def test_dimacs_round_trip(tmp_path, make):
    """write -> read gives the identical network (S:362 round-trip invariant), and the
    parsed instance has the same maximum flow."""
    g = make()
    p = str(tmp_path / "r.max")
    synth.write_dimacs(g, p, comment=g.name)
    h = synth.read_dimacs(p)
    assert (h.n, h.m, h.s, h.t) == (g.n, g.m, g.s, g.t)
    assert np.array_equal(h.row_off, g.row_off)
    assert np.array_equal(h.col, g.col) and np.array_equal(h.cap, g.cap)
    assert not h.meta["arc_count_mismatch"]
    assert oracle.maxflow_graph(h).flow == oracle.maxflow_graph(g).flow


# ------------------------------------------------------------------ SNAP
def test_snap_examples(tmp_path):
    n, s, d, c = synth.read_snap(_w(tmp_path, "a.txt", "# hdr\n3 7\n7 3\n"))
    assert n == 2 and sorted(zip(s.tolist(), d.tolist())) == [(0, 1), (1, 0)] and c.tolist() == [1, 1]
    n, s, d, c = synth.read_snap(_w(tmp_path, "b.txt", "3 7\n3 7\n"))           # cap 2
    assert n == 2 and s.tolist() == [0] and d.tolist() == [1] and c.tolist() == [2]
    n, s, d, c = synth.read_snap(_w(tmp_path, "c.txt", ""))                    # empty
    assert n == 0 and s.size == 0


def test_snap_remap_first_appearance_and_self_loops(tmp_path):
    txt = "# c\n100 5\n5 100\r\n42 42\n5 9000000000\n\t9000000000   100 \n"
    n, s, d, c = synth.read_snap(_w(tmp_path, "a.txt", txt))
    # first appearance: 100 -> 0, 5 -> 1, 42 -> 2, 9000000000 -> 3
    assert n == 4
    assert sorted(zip(s.tolist(), d.tolist())) == [(0, 1), (1, 0), (1, 3), (3, 0)]


def test_snap_malformed(tmp_path):
    with pytest.raises(synth.IngestError) as ei:
        synth.read_snap(_w(tmp_path, "a.txt", "# c\n1 2\n3\n"))
    assert ei.value.code == -4 and ei.value.line == 3


def test_snap_instance_matches_generator_graph(tmp_path):
    """An R-MAT edge list written as a SNAP file with shuffled, sparse ids parses back to an
    isomorphic graph; with the paper's pair rule on top the oracle's F equals scipy's."""
    src, dst, _ = synth.rmat_edges(10, 8, seed=5)
    rng = np.random.default_rng(0)
    ids = rng.choice(10**9, size=1 << 10, replace=False)
    p = tmp_path / "rmat.txt"
    with open(p, "w") as f:
        f.write("# Directed graph\n# FromNodeId\tToNodeId\n")
        for a, b in zip(ids[src], ids[dst]):
            f.write(f"{a}\t{b}\n")
    n, s2, d2, c2 = synth.read_snap(str(p))
    touched = np.unique(np.concatenate([src, dst]))
    assert n == touched.size and s2.size == src.size and (c2 == 1).all()
    # bijection check: the degree multisets agree
    assert sorted(np.bincount(s2, minlength=n).tolist()) == sorted(np.bincount(src, minlength=1 << 10)[touched].tolist())
    g = synth.snap_instance(str(p), npairs=4, nstarts=32, seed=3)
    assert g.n == n + 2 and len(g.meta["sources"]) == 4
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_flow
    es, ed, ec = g.edges()
    A = csr_matrix((ec, (es, ed)), shape=(g.n, g.n))
    assert oracle.maxflow_graph(g).flow == maximum_flow(A, g.s, g.t).flow_value


# ------------------------------------------------------------------ KONECT
def test_konect_examples(tmp_path):
    nL, nR, l, r = synth.read_konect(_w(tmp_path, "a.txt", "% bip\n1 1\n2 1\n"))
    assert (nL, nR) == (2, 1) and sorted(zip(l.tolist(), r.tolist())) == [(0, 0), (1, 0)]
    nL, nR, l, r = synth.read_konect(_w(tmp_path, "b.txt", "% bip unweighted\n1 2 5 1167609600\n"))
    assert (nL, nR) == (1, 2) and l.tolist() == [0] and r.tolist() == [1]


def test_konect_header_sizes_and_duplicates(tmp_path):
    txt = "% bip unweighted\n% 4 5 7\n1 1\n2 3 1.5\n2 3\n3 1\n"
    nL, nR, l, r = synth.read_konect(_w(tmp_path, "a.txt", txt))
    assert (nL, nR) == (5, 7) and l.size == 3     # isolated vertices kept from the header
    n, s, d, c, S, T = matching.network(nL, nR, l, r)
    assert oracle.maxflow_graph(synth.from_edges(n, s, d, c, S, T)).flow == 2   # {(0,0), (1,2)}


def test_konect_malformed(tmp_path):
    with pytest.raises(synth.IngestError) as ei:
        synth.read_konect(_w(tmp_path, "a.txt", "% x\n1 0\n"))
    assert ei.value.code == -5 and ei.value.line == 2


# ------------------------------------------------------------------ the paper's files, when supplied
def _datasets():
    with open(os.path.join(ROOT, "tests", "golden", "paper_datasets.json")) as f:
        return json.load(f)


def _find(name):
    base = os.environ.get("WBPR_DATASETS")
    if not base:
        return None
    for root, _, files in os.walk(base):
        for fn in files:
            if name.lower() in fn.lower():
                return os.path.join(root, fn)
    return None


@pytest.mark.parametrize("row", _datasets()["konect"], ids=lambda r: r["id"])
def test_table2_matching_size(row):
    """Table 2: |L|, |R|, |E| and the maximum matching of each KONECT graph.
    Skipped unless the file is supplied (WBPR_DATASETS=dir)."""
    path = _find(row["name"])
    if path is None:
        pytest.skip(f"{row['name']} not supplied (WBPR_DATASETS)")
    nL, nR, l, r = synth.read_konect(path)
    assert (nL, nR, l.size) == (row["L"], row["R"], row["E"]), row["citation"]
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import maximum_bipartite_matching
    A = csr_matrix((np.ones(l.size, np.int8), (l, r)), shape=(nL, nR))
    assert int((maximum_bipartite_matching(A, perm_type="column") >= 0).sum()) == row["maxflow"], row["citation"]


@pytest.mark.parametrize("row", _datasets()["snap"] + _datasets()["dimacs"], ids=lambda r: r["id"])
def test_table1_sizes(row):
    """Table 1 |V| and |E|; skipped unless the file is supplied."""
    path = _find(row["name"])
    if path is None:
        pytest.skip(f"{row['name']} not supplied (WBPR_DATASETS)")
    if row["id"].startswith("S"):
        g = synth.read_dimacs(path)
        assert (g.n, g.m) == (row["V"], row["E"]), row["citation"]
    else:
        n, s, _, _ = synth.read_snap(path)
        assert n == row["V"], row["citation"]
