import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle
import paper_2404_00270_b200 as W
from oracle import check
from tests.gpu_helpers import dense_bcsr, to_dev
g = synth.grid(40, 30, True, 2)
ref = oracle.maxflow_graph(g, phase2=False)
ro, col, cap = to_dev(g)
ws = W.Workspace(W.workspace_size(g.n, g.m))
try:
    F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, workspace=ws, push_mode=0, bfs_mode=0, small_mode=1, gap_mode=1)
    print("ok", F)
except Exception as e:
    print("ERR", e)
R0 = W.residual(ws)
R = dict(R0, **dense_bcsr(R0))
N = g.n
e = R["e"]; h = R["h"]
print("e(t)", e[g.t], "ref", ref.flow, "sum e", e.sum(), "neg e", (e < 0).sum(), "neg cf", (R["cf"] < 0).sum())
cons = R["cf"] + R["cf"][R["mate"]] - R["cap0"] - R["cap0"][R["mate"]]
print("pair conservation violations", (cons != 0).sum())
# excess vs net flow consistency
owner = np.repeat(np.arange(N), np.diff(R["off"]))
flow_out = np.zeros(N, np.int64)
x = R["cap0"].astype(np.int64) - R["cf"]
np.add.at(flow_out, owner, x)
print("excess mismatch (e != -netout except s)", ((e + flow_out) != 0).sum(), "at s", e[g.s] + flow_out[g.s])
act = (e > 0) & (h < N)
act[[g.s, g.t]] = False
print("active after final GR", act.sum(), "h>=N count", (h >= N).sum())
# reachability to t in residual (BFS on cf>0 arcs reversed)
from collections import deque
reach = np.zeros(N, bool); reach[g.t] = True; dq = deque([g.t])
while dq:
    w = dq.popleft()
    for p in range(R["off"][w], R["off"][w + 1]):
        u = R["col"][p]
        if not reach[u] and R["cf"][R["mate"][p]] > 0:
            reach[u] = True; dq.append(u)
exc = (e > 0); exc[[g.s, g.t]] = False
print("vertices with excess that reach t:", (exc & reach).sum())
print("h consistent with reach (h<N == reach)?", np.array_equal(h < N, reach))
bad = np.nonzero((h < N) != reach)[0][:10]
print("mismatch vertices", bad, h[bad], reach[bad])
