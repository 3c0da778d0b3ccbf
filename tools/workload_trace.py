"""NEXT #3: per-warp workload analysis (§4.3 / Fig. 3) and the Eq. 1
execution-time model (§2.4) on B200, from the device trace (option trace_rounds).

For each graph and schedule (TC = Alg. 1 thread-centric sweeps, VC = Alg. 2 vertex-centric
rounds) it reports, over the traced rounds, the per-warp busy times normalised by their mean
(Fig. 3's measure): the stddev and the max/mean ratio.  It then fits Eq. 1's local-operation
cost  busy_w ~ c0 + k*slots_w + P*pushes_w + R*relabels_w  by non-negative least squares over all warp
records, and checks the model's prediction of each round's time, max_w busy_w (Eq. 1's max).
usage: python tools/workload_trace.py [--rounds 24] > workload_trace.md"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2404_00270_b200 as W


def analyse(recs):
    """recs: structured [rounds, warps]; use warps with work in rounds with work."""
    out = dict(std=[], maxmean=[], rows=[])
    for r in range(recs.shape[0]):
        row = recs[r]
        act = row[(row["tasks"] > 0) | (row["slots"] > 0)]
        if act.shape[0] < 2:
            continue
        b = act["busy_ns"].astype(np.float64)
        mu = b.mean()
        if mu <= 0:
            continue
        out["std"].append(float((b / mu).std()))
        out["maxmean"].append(float(b.max() / mu))
        out["rows"].append(act)
    return out


def fit_eq1(rows):
    X, y = [], []
    for act in rows:
        for a in act:
            X.append([1.0, a["slots"], a["pushes"], a["relabels"]])
            y.append(float(a["busy_ns"]))
    X, y = np.array(X), np.array(y)
    from scipy.optimize import nnls          # Eq. 1's costs k, P, R are non-negative
    coef, _ = nnls(X, y)
    pred_rounds, meas_rounds = [], []
    for act in rows:
        Xa = np.stack([np.ones(act.shape[0]), act["slots"], act["pushes"], act["relabels"]], 1)
        pred_rounds.append(float((Xa @ coef).max()))
        meas_rounds.append(float(act["busy_ns"].max()))
    pr, mr = np.array(pred_rounds), np.array(meas_rounds)
    ss = ((mr - pr) ** 2).sum()
    r2 = 1 - ss / max(((mr - mr.mean()) ** 2).sum(), 1e-9)
    rel = float(np.median(np.abs(pr - mr) / np.maximum(mr, 1)))
    return coef, r2, rel


def fit_rounds(rows):
    """Eq. 1 at the level it is stated: a round's time is the max over tiles of the
    summed local-operation costs, plus a fixed per-round term (barrier, launch of the round's
    dependent memory chain) that the warp-level fit cannot see.  Regress each round's measured
    time (max busy_ns over its warps) on c0 + k * slots_w* + P * pushes_w* + R * relabels_w*,
    where w* is the round's most loaded warp by slots (non-negative least squares, leave-one-out
    R^2 so the intercept cannot fit noise)."""
    from scipy.optimize import nnls
    X, y = [], []
    for act in rows:
        w = int(np.argmax(act["slots"]))
        X.append([1.0, act["slots"][w], act["pushes"][w], act["relabels"][w]])
        y.append(float(act["busy_ns"].max()))
    X, y = np.array(X, np.float64), np.array(y)
    coef, _ = nnls(X, y)
    if len(y) < 4:
        return coef, float("nan")
    pred = np.empty_like(y)
    for i in range(len(y)):
        m = np.ones(len(y), bool)
        m[i] = False
        c, _ = nnls(X[m], y[m])
        pred[i] = X[i] @ c
    r2 = 1 - ((y - pred) ** 2).sum() / max(((y - y.mean()) ** 2).sum(), 1e-9)
    return coef, float(r2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=24)
    a = ap.parse_args()
    graphs = [("R-MAT-18 hub20 (skewed)", synth.rmat(18, 16, 1000, "hub20")),
              ("R-MAT-18 paper rule", synth.rmat(18, 16, 1000, "paper")),
              ("grid 256x256 U[1,100] (road-like)", synth.grid(256, 256, True, 1))]
    print("| graph | schedule | traced rounds | busy/mean stddev (median) | max/mean (median) | "
          "Eq.1 k ns/slot | P ns/push | R ns/relabel | Eq.1 round-time R^2 | median rel. err | "
          "round-level fit c0 us / k ns/slot | round-level LOO R^2 |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name, g in graphs:
        ro, col, cap = (torch.from_numpy(x).cuda() for x in (g.row_off, g.col, g.cap))
        for sch in ("tc", "vc"):
            opt = W.options("bcsr", schedule=sch, trace_rounds=a.rounds, small_mode=0)
            ws = W.Workspace(W.workspace_size(g.n, g.m, 1, opt))
            W.maxflow(ro, col, cap, g.s, g.t, workspace=ws, schedule=sch, trace_rounds=a.rounds, small_mode=0)
            rec = W.trace(ws)
            an = analyse(rec)
            if not an["rows"]:
                continue
            coef, r2, rel = fit_eq1(an["rows"])
            rc, rr2 = fit_rounds(an["rows"])
            print(f"| {name} | {sch.upper()} | {len(an['rows'])} | {np.median(an['std']):.3f} | "
                  f"{np.median(an['maxmean']):.2f} | {coef[1]:.2f} | {coef[2]:.1f} | {coef[3]:.1f} | {r2:.3f} | {rel:.3f} | "
                  f"{rc[0] / 1e3:.2f} / {rc[1]:.2f} | {rr2:.3f} |", flush=True)


if __name__ == "__main__":
    main()
