#!/usr/bin/env python
"""Same-capture DRAM traffic of the solve kernel (run on the GPU box, 1 GPU).

    python tools/traffic_run.py --workload c5 [--layout bcsr] [--out profiles/r2/traffic_c5_bcsr.json]

Runs bench.py under ncu with only the k_solve launches profiled and a metric set that fits one
replay pass (DRAM bytes, duration, L2 hit rate, warp-execution efficiency, occupancy), while
bench.py dumps every step's own device counters (--dump-steps).  Launch i of k_solve is step i
(warm-up included), so each launch's DRAM bytes are divided by the algorithmic bytes of THAT
launch (bench.solve_bytes of its counters): a like-for-like traffic / algorithmic ratio even
though the lock-free trajectory (and with it the work) varies from run to run.  ncu's own
timing is cold-cache and serialised; the ratio, not the duration, is the product here.
bench.py reads the result as roofline.traffic / traffic_same_capture."""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if "k_solve" not in d["Kernel Name"]:
            continue
        i = int(d["ID"])
        v = float(d["Metric Value"].replace(",", ""))
        out.setdefault(i, {})[d["Metric Name"]] = v * SCALE.get(d["Metric Unit"], 1.0)
    return [out[k] for k in sorted(out)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--layout", default="bcsr")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--opt", action="append", default=[])
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = f"{a.workload}_{a.layout}"
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{tag}.csv")
    dump = os.path.join(ROOT, "gpurun_out", f"steps_{tag}.json")
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:k_solve", "--csv",
           "--log-file", log, sys.executable, os.path.join(ROOT, "bench.py"), "--workload", a.workload,
           "--layout", a.layout, "--steps", str(a.steps), "--warmup", "3", "--no-cpu-baseline", "--no-per-graph",
           "--e2e-streams", "0", "--dump-steps", dump] + sum((["--opt", o] for o in a.opt), [])
    r = subprocess.run(cmd, capture_output=True, text=True)
    passes = re.findall(r"(\d+) pass", r.stdout + r.stderr)
    if r.returncode != 0:
        print(r.stdout[-3000:], r.stderr[-3000:])
        sys.exit(r.returncode)
    launches = parse(log)
    steps = json.load(open(dump + ".rank0"))
    if len(launches) != len(steps):
        sys.exit(f"{len(launches)} k_solve launches profiled but {len(steps)} steps dumped")
    per = []
    for L, s in zip(launches, steps):
        dram = L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"]
        per.append({"dram_bytes": int(dram), "algorithmic_bytes": int(s["solve_bytes"]),
                    "ratio": round(dram / s["solve_bytes"], 4), "ncu_ms": round(L["gpu__time_duration.sum"], 3),
                    "l2_hit_pct": round(L.get("lts__t_sector_hit_rate.pct", 0.0), 2),
                    "warp_efficiency": round(L.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0.0) / 32, 4),
                    "occupancy_pct": round(L.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0), 2),
                    "bfs_arcs_scanned": s["bfs_arcs_scanned"], "bfs_arcs_bottom_up": s["bfs_arcs_bottom_up"],
                    "arcs_scanned": s["arcs_scanned"], "rounds": s["rounds"], "global_relabels": s["global_relabels"]})
    med = sorted(per, key=lambda x: x["ratio"])[len(per) // 2]
    res = {"workload": a.workload, "layout": a.layout, "launches": len(per), "replay_passes_seen": sorted(set(passes)),
           "dram_bytes_per_launch": med["dram_bytes"], "algorithmic_bytes_per_launch": med["algorithmic_bytes"],
           "ratio": med["ratio"], "l2_hit_pct": med["l2_hit_pct"], "warp_efficiency": med["warp_efficiency"],
           "occupancy_pct": med["occupancy_pct"],
           "source": "ncu --metrics " + ",".join(METRICS) + " -k regex:k_solve, every launch paired with the "
                     "counters of the same launch (bench.py --dump-steps); median launch by ratio",
           "per_launch": per}
    out = a.out or os.path.join(ROOT, "gpurun_out", f"traffic_{tag}.json")   # copied to profiles/r2/ by hand
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}))


if __name__ == "__main__":
    main()
