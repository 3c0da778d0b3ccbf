"""Time the A1 construction alone (wbpr_build_residual) on a workload: median build_ms of N runs.
usage: python tools/build_time.py [c5|c3|c4net] [--reps 5]   (WBPR_LIB selects an experiment build)"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2404_00270_b200 as W
ap = argparse.ArgumentParser(); ap.add_argument("wl", nargs="?", default="c5"); ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
if a.wl == "c5":
    import json as _j
    B = synth.disjoint_union(synth.c5_batch(64))
    g = B.union
elif a.wl == "c3":
    g = synth.rmat(22, 16, 1, "paper")
else:
    g = synth.rmat(18, 16, 1000, "paper")
ro, col, cap = (torch.from_numpy(x).cuda() for x in (g.row_off, g.col, g.cap))
ws = W.Workspace(W.workspace_size(g.n, g.m, 1, W.options("bcsr")))
ms = []
for i in range(a.reps + 2):
    _, st = W.build_residual(ro, col, cap, "bcsr", workspace=ws)
    if i >= 2: ms.append(st["build_ms"])
print(json.dumps({"wl": a.wl, "lib": os.environ.get("WBPR_LIB", "default"), "build_ms": float(np.median(ms)), "M": st["M"]}))
