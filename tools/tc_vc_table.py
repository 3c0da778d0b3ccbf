"""B200 analogue of the paper's Tables 1-2: thread-centric (TC, Alg. 1) vs vertex-centric
(VC, Alg. 2) x BCSR / RCSR solve times on the synthetic configs, median of R runs.
usage: python tools/tc_vc_table.py [--reps 3] [cfg ...]  -> markdown on stdout"""
import argparse, json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="*", default=["c2u", "c2r", "c3p", "c3h", "c4", "r18p", "r18h"])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
res = {}
for sch in ("vc", "tc"):
    for lay in ("rcsr", "bcsr"):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "probe.py"), *a.cfgs, "--reps", str(a.reps),
                              "--schedule", sch, "--layout", lay], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            try:
                d = json.loads(ln)
            except Exception:
                continue
            if "solve_ms" in d:
                res.setdefault((d["cfg"], sch, lay), []).append(d)
print("| config | VC+RCSR ms | VC+BCSR ms | TC+RCSR ms | TC+BCSR ms | TC/VC RCSR | TC/VC BCSR | F |")
print("|---|---|---|---|---|---|---|---|")
for c in a.cfgs:
    def med(s, l):
        v = [d["solve_ms"] for d in res.get((c, s, l), [])]
        return float(np.median(v)) if v else float("nan")
    vr, vb, tr, tb = med("vc", "rcsr"), med("vc", "bcsr"), med("tc", "rcsr"), med("tc", "bcsr")
    F = res.get((c, "vc", "bcsr"), [{}])[0].get("flow_value")
    print(f"| {c} | {vr:.2f} | {vb:.2f} | {tr:.2f} | {tb:.2f} | {tr / vr:.2f}x | {tb / vb:.2f}x | {F} |")
