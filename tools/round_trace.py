"""Per-round straggler view of the VC rounds (device trace, option trace_rounds).
For each traced round: active warps, mean / max warp busy time, and the slowest warp's
tasks / slots / pushes / relabels.   usage: python tools/round_trace.py c5|r18h|c3h [--rounds 64]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2404_00270_b200 as W

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--rounds", type=int, default=64)
a = ap.parse_args()
opt = dict(trace_rounds=a.rounds)
if a.cfg == "c5":
    B = synth.disjoint_union(synth.c5_batch())
    G = B.union
    ro, col, cap = (torch.from_numpy(x).cuda() for x in (G.row_off, G.col, G.cap))
    ws = W.Workspace(W.workspace_size(G.n, G.m, 64, W.options("bcsr", **opt)))
    for _ in range(2):
        _, _, _, st = W.maxflow_batch(ro, col, cap, B.vbase, B.s, B.t, workspace=ws, **opt)
else:
    def c4():
        from oracle import matching
        l, r = synth.bipartite_edges()
        n, src, dst, cap, s_, t_ = matching.network(1 << 20, 1 << 20, l, r)
        return synth.from_edges(n, src, dst, cap, s_, t_)
    g = {"r18h": lambda: synth.rmat(18, 16, 1000, "hub20"), "c3h": lambda: synth.rmat(22, 16, 1, "hub20"),
         "c3p": lambda: synth.rmat(22, 16, 1, "paper"), "c4": c4}[a.cfg]()
    ro, col, cap = (torch.from_numpy(x).cuda() for x in (g.row_off, g.col, g.cap))
    ws = W.Workspace(W.workspace_size(g.n, g.m, 1, W.options("bcsr", **opt)))
    for _ in range(2):
        _, _, st = W.maxflow(ro, col, cap, g.s, g.t, workspace=ws, **opt)
rec = W.trace(ws)
print(f"rounds {st['rounds']} solve_ms {st['solve_ms']:.2f} round phases ms {st['phase_ns'][1] / 1e6:.2f}")
print("round act_warps mean_us max_us | slowest: tasks slots pushes relabels | p99_us  sum_slots")
for r in range(rec.shape[0]):
    row = rec[r]
    act = row[(row["tasks"] > 0)]
    if act.shape[0] == 0:
        continue
    b = act["busy_ns"].astype(np.float64) / 1e3
    i = int(np.argmax(b))
    s = act[i]
    print(f"{r:4d} {act.shape[0]:6d} {b.mean():8.2f} {b.max():8.2f} | {s['tasks']:4d} {s['slots']:7d} {s['pushes']:5d} "
          f"{s['relabels']:4d} | {np.percentile(b, 99):8.2f} {int(act['slots'].sum()):9d}")
