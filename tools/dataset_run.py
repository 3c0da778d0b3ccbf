"""Run a dataset file end to end on the GPU and check it against the oracle (NEXT #4).

    python tools/dataset_run.py FILE [--format dimacs|snap|konect] [--layout bcsr|rcsr]
                                     [--pairs 20] [--seed 1] [--no-oracle]

DIMACS files use their own s/t; SNAP edge lists get the paper's 20 BFS-selected pairs behind a
super-source and super-sink; KONECT bipartite lists run through the matching
wrapper, and the size is compared with Table 2 when the file name matches a
row of tests/golden/paper_datasets.json.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("file")
    ap.add_argument("--format", choices=["dimacs", "snap", "konect"])
    ap.add_argument("--layout", default="bcsr", choices=["bcsr", "rcsr"])
    ap.add_argument("--pairs", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    fmt = a.format or ("dimacs" if a.file.endswith((".max", ".dimacs")) else
                       "konect" if "konect" in a.file or a.file.startswith("out.") else "snap")
    import torch
    import paper_2404_00270_b200 as W
    t0 = time.perf_counter()
    rec = {"file": os.path.basename(a.file), "format": fmt, "layout": a.layout}
    if fmt == "konect":
        nL, nR, l, r = synth.read_konect(a.file)
        rec.update(nL=nL, nR=nR, E=int(l.size), ingest_s=round(time.perf_counter() - t0, 3))
        size, match, st = W.bipartite_match(nL, nR, torch.from_numpy(l).cuda(), torch.from_numpy(r).cuda(),
                                            layout=a.layout)
        rec.update(matching=size, solve_ms=st["solve_ms"], build_ms=st["build_ms"])
        if not a.no_oracle:
            import oracle
            from oracle import matching
            n, s, d, c, S, T = matching.network(nL, nR, l, r)
            F = oracle.maxflow_graph(synth.from_edges(n, s, d, c, S, T), phase2=False).flow
            matching.check_matching(nL, nR, l, r, match.cpu().numpy(), size)
            rec.update(oracle_flow=F, parity=F == size)
        with open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "paper_datasets.json")) as f:
            for row in json.load(f)["konect"]:
                if row["name"].lower() in a.file.lower():
                    rec.update(table2=row["maxflow"], table2_match=row["maxflow"] == size, cite=row["citation"])
    else:
        g = synth.read_dimacs(a.file) if fmt == "dimacs" else synth.snap_instance(a.file, a.pairs, 256, a.seed)
        rec.update(n=g.n, m=g.m, ingest_s=round(time.perf_counter() - t0, 3))
        ro, col, cap = (torch.from_numpy(x).cuda() for x in (g.row_off, g.col, g.cap))
        F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, layout=a.layout)
        rec.update(flow=F, cut_capacity=st["cut_capacity"], solve_ms=st["solve_ms"], build_ms=st["build_ms"],
                   rounds=st["rounds"], global_relabels=st["global_relabels"])
        if not a.no_oracle:
            import oracle
            ref = oracle.maxflow_graph(g, phase2=False)
            rec.update(oracle_flow=ref.flow, parity=bool(ref.flow == F and np.array_equal(
                bm.cpu().numpy().view(np.uint32), ref.bitmap_words())))
    print(json.dumps(rec))
    return 0 if rec.get("parity", True) else 1


if __name__ == "__main__":
    sys.exit(main())
