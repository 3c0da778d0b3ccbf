"""Quick GPU probe: solve a list of configs through the C-ABI, print stats JSON lines.
usage: python tools/probe.py c1 c2u c2r c3p c3h c4 [--layout bcsr|rcsr] [--beta B]"""
import argparse, json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2404_00270_b200 as W


def graph(name):
    if name == "c1": return synth.random_graph(1024, 8192, 1)
    if name == "c2u": return synth.grid(1024, 1024, False, 1)
    if name == "c2r": return synth.grid(1024, 1024, True, 1)
    if name == "g256r": return synth.grid(256, 256, True, 1)
    if name == "g128r": return synth.grid(128, 128, True, 1)
    if name == "r14p": return synth.rmat(14, 16, 1, "paper")
    if name == "r14h": return synth.rmat(14, 16, 1, "hub20")
    if name == "rand16k": return synth.random_graph(16384, 131072, 1, 0, 16383)
    if name == "c3p": return synth.rmat(22, 16, 1, "paper")
    if name == "c3h": return synth.rmat(22, 16, 1, "hub20")
    if name == "r18p": return synth.rmat(18, 16, 1000, "paper")
    if name == "r18h": return synth.rmat(18, 16, 1000, "hub20")
    if name == "rlg": return synth.washington_rlg()
    if name == "genrmf": return synth.genrmf()
    if name.startswith("path"):
        k = int(name[4:])
        src = np.arange(k - 1); dst = src + 1
        return synth.from_edges(k, src, dst, np.ones(k - 1, np.int32), 0, k - 1, name=name)
    raise ValueError(name)


ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="+")
ap.add_argument("--layout", default="bcsr")
ap.add_argument("--beta", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--blocks", type=int, default=0)
ap.add_argument("--mode", type=int, default=1)
ap.add_argument("--gamma", type=float, default=-1.0)
ap.add_argument("--persist", type=int, default=0)
ap.add_argument("--bfs", type=int, default=1)
ap.add_argument("--small", type=int, default=1)
ap.add_argument("--gap", type=int, default=0)
ap.add_argument("--schedule", default="vc")
ap.add_argument("--groups", type=int, default=0)
ap.add_argument("--oracle", action="store_true")
a = ap.parse_args()
for name in a.cfgs:
    t0 = time.time()
    if name == "c5":
        B = synth.disjoint_union(synth.c5_batch())
        G = B.union
        ro, col, cap = (torch.from_numpy(x).cuda() for x in (G.row_off, G.col, G.cap))
        opt = W.options(a.layout)
        ws = W.Workspace(W.workspace_size(G.n, G.m, 64, opt))
        gen = time.time() - t0
        for rep in range(a.reps):
            flows, cuts, bm, st = W.maxflow_batch(ro, col, cap, B.vbase, B.s, B.t, layout=a.layout, workspace=ws,
                                                  gr_beta=a.beta, timeout_ms=100000, grid_blocks=a.blocks,
                                                  push_mode=a.mode, gr_gamma=a.gamma, l2_persist=a.persist,
                                                  bfs_mode=a.bfs, small_mode=a.small, gap_mode=a.gap,
                                                  schedule=a.schedule, batch_groups=a.groups)
            print(json.dumps(dict(cfg=name, rep=rep, gen_s=round(gen, 2), **st)), flush=True)
        continue
    if name == "c4":
        l, r = synth.bipartite_edges()
        lt, rt = torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda()
        gen = time.time() - t0
        for rep in range(a.reps):
            size, match, st = W.bipartite_match(1 << 20, 1 << 20, lt, rt, layout=a.layout, gr_beta=a.beta,
                                                timeout_ms=100000, grid_blocks=a.blocks, push_mode=a.mode, gr_gamma=a.gamma, l2_persist=a.persist, bfs_mode=a.bfs, small_mode=a.small, gap_mode=a.gap, schedule=a.schedule)
            print(json.dumps(dict(cfg=name, rep=rep, gen_s=round(gen, 2), size=size, **st)), flush=True)
        continue
    g = graph(name)
    gen = time.time() - t0
    ro, col, cap = (torch.from_numpy(x).cuda() for x in (g.row_off, g.col, g.cap))
    ws = W.Workspace(W.workspace_size(g.n, g.m, 1, W.options(a.layout)))
    for rep in range(a.reps):
        F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, layout=a.layout, workspace=ws, gr_beta=a.beta,
                              timeout_ms=100000, grid_blocks=a.blocks, push_mode=a.mode, gr_gamma=a.gamma, l2_persist=a.persist, bfs_mode=a.bfs, small_mode=a.small, gap_mode=a.gap, schedule=a.schedule)
        print(json.dumps(dict(cfg=name, rep=rep, gen_s=round(gen, 2), **st)), flush=True)
    if a.oracle:
        import oracle
        r = oracle.maxflow_graph(g, phase2=False)
        print(json.dumps(dict(cfg=name, oracle_flow=r.flow, oracle_s=r.seconds,
                              bitmap_equal=bool(np.array_equal(bm.cpu().numpy().view(np.uint32), r.bitmap_words())))),
              flush=True)
