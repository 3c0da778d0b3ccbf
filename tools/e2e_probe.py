"""How much of a C5 step's H2D copy overlaps another step's kernels?  Times (a) the pinned
H2D of the union CSR alone, (b) one device-resident solve alone, (c) both issued together on
two streams (copy into a scratch device buffer)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2404_00270_b200 as W

B = synth.disjoint_union(synth.c5_batch())
G = B.union
dev = torch.device("cuda", 0)
ro_h, col_h, cap_h = (torch.from_numpy(x).pin_memory() for x in (G.row_off, G.col, G.cap))
ro_d, col_d, cap_d = (x.to(dev) for x in (ro_h, col_h, cap_h))
scratch = [torch.empty_like(x, device=dev) for x in (ro_h, col_h, cap_h)]
ws = W.Workspace(W.workspace_size(G.n, G.m, 64, W.options("bcsr")), dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

def copy():
    with torch.cuda.stream(s1):
        for d, h in zip(scratch, (ro_h, col_h, cap_h)):
            d.copy_(h, non_blocking=True)

def solve():
    with torch.cuda.stream(s2):
        W.maxflow_batch(ro_d, col_d, cap_d, B.vbase, B.s, B.t, workspace=ws, device=dev, gr_gamma=0.5)

for f in (copy, solve):
    f(); torch.cuda.synchronize()
for name, fs in (("copy", [copy]), ("solve", [solve]), ("both", [copy, solve])):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ths = [threading.Thread(target=f) for f in fs]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t0) * 1e3, 2), "ms", flush=True)
