"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck), each
checked against the oracle so a sanitizer run is also a parity run:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

C1 (random 1K / 8K) on both layouts and both schedules, a 32x32 random-capacity grid, a 3-
instance batch, a bipartite matching, phase 2 and the online gap, with a long device watchdog
(the sanitizer slows the persistent kernel by orders of magnitude)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2404_00270_b200 as W  # noqa: E402
from oracle import matching  # noqa: E402

TMO = 600000


def run(g, **opt):
    ro, col, cap = (torch.from_numpy(a).cuda() for a in (g.row_off, g.col, g.cap))
    F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, timeout_ms=TMO, **opt)
    ref = oracle.maxflow_graph(g, phase2=False)
    ok = F == ref.flow and np.array_equal(bm.cpu().numpy().view(np.uint32), ref.bitmap_words())
    print(f"{g.name} {opt}: F={F} oracle={ref.flow} {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    which = sys.argv[1:] or ["c1", "grid", "batch", "bip", "modes"]
    ok = True
    c1 = synth.random_graph(1024, 8192, 1)
    if "c1" in which:
        for layout in ("bcsr", "rcsr"):
            ok &= run(c1, layout=layout)          # (BCSR: the one-CTA tiny path)
        ok &= run(c1, tiny_mode=1)                # the multi-kernel path on the same instance
        ok &= run(c1, schedule="tc")
    if "grid" in which:
        ok &= run(synth.grid(32, 32, True, 3))
    if "modes" in which:
        ok &= run(c1, phase2=1)
        ok &= run(c1, gap_mode=1)
        ok &= run(c1, push_mode=0)
    if "batch" in which:
        parts = [synth.random_graph(300, 2000, i, 0, 299) for i in range(3)]
        B = synth.disjoint_union(parts)
        ro, col, cap = (torch.from_numpy(a).cuda() for a in (B.union.row_off, B.union.col, B.union.cap))
        flows, cuts, _, _ = W.maxflow_batch(ro, col, cap, B.vbase, B.s, B.t, timeout_ms=TMO)
        good = all(flows[i] == oracle.maxflow_graph(p, phase2=False).flow == cuts[i] for i, p in enumerate(parts))
        print(f"batch3: {list(flows)} {'OK' if good else 'MISMATCH'}", flush=True)
        ok &= good
    if "bip" in which:
        l, r = synth.bipartite_edges(200, 150, 500, 1)
        size, match, _ = W.bipartite_match(200, 150, torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda(),
                                           timeout_ms=TMO)
        n, s, d, c, S, T = matching.network(200, 150, l, r)
        F = oracle.maxflow_graph(synth.from_edges(n, s, d, c, S, T), phase2=False).flow
        matching.check_matching(200, 150, l, r, match.cpu().numpy(), size)
        print(f"bipartite: {size} oracle={F} {'OK' if size == F else 'MISMATCH'}", flush=True)
        ok &= size == F
    torch.cuda.synchronize()
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
