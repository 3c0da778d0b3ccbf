"""Debug helper: build the BCSR of a graph on the GPU and list vertices whose segment differs
from the reference layout (oracle/residual_ref), with their chunk-relative positions."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2404_00270_b200 as W
from oracle import residual_ref
from tests.gpu_helpers import dense_bcsr

kind = sys.argv[1] if len(sys.argv) > 1 else "c1"
g = synth.shuffle_rows(synth.random_graph(1024, 8192, 1), 1) if kind == "c1" else synth.rmat(int(kind), 16, 1, "paper")
ro, col, cap = (torch.from_numpy(a).cuda() for a in (g.row_off, g.col, g.cap))
ws = W.Workspace(W.workspace_size(g.n, g.m, 1, W.options("bcsr")))
G, st = W.build_residual(ro, col, cap, "bcsr", workspace=ws)
R = W.residual(ws)
seg = R["seg"].astype(np.int64)
ref = residual_ref.bcsr(g.n, g.row_off, g.col, g.cap)
reflen = np.diff(ref["off"])
lens = seg[:, 1] - seg[:, 0]
src, dst, _ = g.edges()
outd = np.diff(g.row_off); ind = np.bincount(dst[src != dst], minlength=g.n)
start = np.concatenate([[0], np.cumsum(outd)])[:-1] + np.concatenate([[0], np.cumsum(ind)])[:-1]
bad = np.nonzero(lens != reflen)[0]
out = {"kind": kind, "M": int(st["M"]), "refM": int(ref["col"].shape[0]), "nbad": int(bad.size), "bad": []}
for x in bad[:40]:
    out["bad"].append(dict(x=int(x), len=int(lens[x]), ref=int(reflen[x]), seg0=int(seg[x, 0]), start=int(start[x]),
                           lo=int(outd[x]), li=int(ind[x]), rel=int(start[x] % 2048)))
print(json.dumps(out))
