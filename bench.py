#!/usr/bin/env python
"""bench.py — WBPR max-flow hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c1|c2|c2r|c3|c3h|c4]
                    [--layout bcsr|rcsr] [--impl wbpr|reference]

One step = one pass of the whole hot path (§8(a) A1-A8, A10: device residual
construction, preflow, push/relabel rounds with device global relabels and
termination, result extraction) over one batch of synthetic input resident in
HBM, through the C-ABI (libwbpr.so).  Default workload (every N): BASELINE.json
configs[4] "C5" — 64 independent R-MAT scale-18 max-flow instances (paper-rule
terminals) partitioned over the N ranks (one process per GPU), solved per rank as
one disjoint-union batch, results gathered with NCCL all_gather.  value = whole-
job instances/s.  Per-graph workloads (C1-C4) are available with --workload.

--impl reference: the CPU oracle (oracle/, FIFO push-relabel + gap, single
thread) timed on this host as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max-flow solve ms & residual GTEPS per graph (1 B200); batch instances/s at 1/2/4/8"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")

# Algorithmic bytes per unit of work (restated in DESIGN.md)
B_SLOT = 12        # scanned residual slot: col 4 + cf 4 + h[col] 4
B_VERTEX = 32      # processed active vertex: queue 4 + 2 offsets 8 + e 8 + h 4 (+ bookkeeping)
B_PUSH = 52        # mate 4 + two cf RMW 16 + two e RMW 32
B_RELABEL = 4
B_BFS_ARC = 16     # top-down: col 4 + mate 4 + cf[mate] 4 + h[u] 4
B_GR_VERTEX = 8    # label reset + write per vertex per global relabel
B_CAND = 12        # compaction candidate: e 8 + h 4


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------- workloads
# Solver options the bench uses per workload unless --opt overrides them (wbpr_options
# fields).  C5: a global relabel after 0.5x (instead of 1x) the last GR's
# time in rounds - measured best on C5 (γ sweep in profiles/r1/); results are exact for
# every γ, it only moves time between rounds and global relabels.
WORKLOAD_OPTS = {"c5": {"gr_gamma": 0.5}}
def make_workload(name, rank, world):
    """Returns dict(kind, parts|graph, ids, desc) for this rank."""
    import synth
    if name == "c5":
        from paper_2404_00270_b200.batch import partition
        total = 64
        lo, hi = partition(total, world, rank)
        parts = [synth.rmat(18, 16, 1000 + i, "paper") for i in range(lo, hi)]
        return dict(kind="batch", parts=parts, ids=list(range(lo, hi)), total=total,
                    desc="C5: 64 x R-MAT scale 18 (edgefactor 16, U[1,100] caps, 20 paper-rule s/t pairs "
                         "behind super terminals), seeds 1000-1063, partitioned over ranks")
    if name == "c4":
        nL = nR = 1 << 20
        l, r = synth.bipartite_edges(nL, nR, 1 << 24, 1)
        return dict(kind="bipartite", nL=nL, nR=nR, l=l, r=r, ids=[rank], total=1,
                    desc="C4: bipartite matching 2^20 x 2^20, 2^24 uniform draws (duplicates collapsed), unit "
                         "capacities via super source/sink (network built on the device, A9)")
    g = {"c1": lambda: synth.random_graph(1024, 8192, 1),
         "c2": lambda: synth.grid(1024, 1024, False, 1),
         "c2r": lambda: synth.grid(1024, 1024, True, 1),
         "c3": lambda: synth.rmat(22, 16, 1, "paper"),
         "c3h": lambda: synth.rmat(22, 16, 1, "hub20")}[name]()
    return dict(kind="single", graph=g, ids=[rank], total=1, desc=g.name)


def union_of(parts):
    import synth
    return synth.disjoint_union(parts)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- roofline
def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def solve_bytes(st):
    """Algorithmic bytes moved by one launch of the persistent solve kernel."""
    return (B_SLOT * st["arcs_scanned"] + B_VERTEX * st["avq_total"] + B_PUSH * st["pushes"] +
            B_RELABEL * st["relabels"] + B_BFS_ARC * st["bfs_arcs_scanned"] +
            B_GR_VERTEX * st["n"] * st["global_relabels"] + B_CAND * st["compaction_candidates"])


def build_bytes(st):
    """Algorithmic bytes of construction A1 (BCSR, merge build): read the input CSR
    (8 B/edge + 8 B/row), write+read the 8-B out-keys and the 4-B in-list entries once,
    write 16 B per output slot (arc 8 + mate 4 + cap0 4)."""
    m, n, M = st["m"], st["n"], st["M"]
    return 8 * m + 8 * n + 2 * 8 * m + 2 * 4 * m + 16 * M


# ---------------------------------------------------------------------------- wbpr arm
def run_wbpr(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2404_00270_b200 as W

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    t0 = time.time()
    wl = make_workload(args.workload, rank, world)
    gen_s = time.time() - t0
    if wl["kind"] == "bipartite":
        return run_bipartite(args, rank, world, dev, wl, gen_s)
    if wl["kind"] == "batch":
        B = union_of(wl["parts"])
        G = B.union
        vbase, s, t = B.vbase, B.s, B.t
    else:
        G = wl["graph"]
        vbase, s, t = np.array([0, G.n]), np.array([G.s]), np.array([G.t])
    k = len(s)
    ro_d = torch.from_numpy(G.row_off).to(dev)
    col_d = torch.from_numpy(G.col).to(dev)
    cap_d = torch.from_numpy(G.cap).to(dev)
    ro_h = torch.from_numpy(G.row_off).pin_memory()
    col_h = torch.from_numpy(G.col).pin_memory()
    cap_h = torch.from_numpy(G.cap).pin_memory()
    opt = dict(layout=args.layout, **WORKLOAD_OPTS.get(args.workload, {}))
    for kv in args.opt:
        k_, v_ = kv.split("=")
        opt[k_] = float(v_) if "." in v_ else int(v_)
    ws = W.Workspace(W.workspace_size(G.n, G.m, k, W.options(args.layout)), dev)
    bitmap_d = torch.empty((G.n + 31) // 32, dtype=torch.int32, device=dev)
    bitmap_h = torch.empty((G.n + 31) // 32, dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream(dev)
    from paper_2404_00270_b200.batch import gather_records, make_records
    gathered = None

    def step(host=False):
        if host:
            flows, cuts, _, st = W.maxflow_batch(ro_h, col_h, cap_h, vbase, s, t, workspace=ws, bitmap=bitmap_h,
                                                 device=dev, **opt)
        else:
            flows, cuts, _, st = W.maxflow_batch(ro_d, col_d, cap_d, vbase, s, t, workspace=ws, bitmap=bitmap_d,
                                                 device=dev, **opt)
        # 64-B result record per instance (id, status, F, cut, rounds, GRs, pushes, relabels),
        # gathered over ranks: the only collective (NCCL all_gather)
        nonlocal gathered
        rec = torch.from_numpy(make_records(wl["ids"], flows, cuts, st)).to(dev)
        gathered = gather_records(rec, wl["total"] if wl["kind"] == "batch" else world, world)
        return st, flows, cuts

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local_rank)
    clk.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sts = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0.record(stream)
    for _ in range(args.steps):
        st, flows, cuts = step()
        sts.append(st)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    # e2e: same metric through the C-ABI with HOST buffers (H2D of the pinned CSR + D2H of the
    # bitmap inside every step).  Steps are issued by `args.e2e_streams` host threads, each with
    # its own stream and workspace (the public API used concurrently), so one step's H2D copy
    # overlaps another step's kernels; timed by wall clock between two device synchronizations.
    # (--e2e-streams 0: no e2e leg - profiler runs whose last step must be a device-resident one)
    e2e_steps = max(1, min(args.steps, 5)) if args.e2e_streams <= 1 else max(2 * args.e2e_streams, min(args.steps, 8))
    pipes = []
    for _ in range(max(1, args.e2e_streams)):
        pipes.append(dict(stream=torch.cuda.Stream(dev), ws=ws if not pipes else
                          W.Workspace(W.workspace_size(G.n, G.m, k, W.options(args.layout)), dev),
                          bm=torch.empty((G.n + 31) // 32, dtype=torch.int32).pin_memory()))

    def host_steps(pp, count):
        torch.cuda.set_device(dev)
        with torch.cuda.stream(pp["stream"]):
            for _ in range(count):
                W.maxflow_batch(ro_h, col_h, cap_h, vbase, s, t, workspace=pp["ws"], bitmap=pp["bm"], device=dev,
                                **opt)

    if args.e2e_streams <= 0:
        pipes = pipes[:0]
    for pp in pipes:            # warm each pipe once (workspace / stream first use)
        host_steps(pp, 1)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    if not pipes:
        pass
    elif len(pipes) == 1:
        host_steps(pipes[0], e2e_steps)
    else:
        per = [e2e_steps // len(pipes) + (1 if i < e2e_steps % len(pipes) else 0) for i in range(len(pipes))]
        ths = [threading.Thread(target=host_steps, args=(pp, c)) for pp, c in zip(pipes, per)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    torch.cuda.synchronize(dev)
    e2e_ms = (time.perf_counter() - t0) * 1e3
    del pipes
    times = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(times[0]), float(times[1])
    total_units = wl["total"] if wl["kind"] == "batch" else world
    value = total_units * args.steps / (ms / 1e3)
    e2e_value = total_units * e2e_steps / (e2e_ms / 1e3) if args.e2e_streams > 0 else None
    if rank != 0:
        return None
    # certificate of every gathered record: F == cut capacity
    g = gathered.cpu().numpy()
    assert np.all(g[:, 2] == g[:, 3]), "certificate failed in gathered records"
    assert np.all(flows == cuts)
    # roofline of the dominant kernel: the persistent solve kernel k_solve (the largest single
    # launch of every step, profiles/); the construction kernels are reported beside it
    hbm, peak_src = peaks()
    solve_ms = float(np.mean([x["solve_ms"] for x in sts]))
    build_ms = float(np.mean([x["build_ms"] for x in sts]))
    total_ms = float(np.mean([x["total_ms"] for x in sts]))
    st = sts[-1]
    sb, bb = solve_bytes(st), build_bytes(st)
    achieved = sb / (solve_ms / 1e3) / 1e9
    build_achieved = bb / (build_ms / 1e3) / 1e9
    gteps = (st["arcs_scanned"] + st["bfs_arcs_scanned"]) / (solve_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{args.workload}:{args.layout}")
        except Exception:
            traffic = None
    h2d = int(G.row_off.nbytes + G.col.nbytes + G.cap.nbytes)
    d2h = int(bitmap_h.numel() * 4 + 16 * k)
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "instances/s" if wl["kind"] == "batch" else "solves/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "strong" if wl["kind"] == "batch" else "weak",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "layout": args.layout,
                   "options": {k_: v_ for k_, v_ in opt.items() if k_ != "layout"},
                   "instances_per_rank": k, "n_per_rank": int(G.n), "m_per_rank": int(G.m),
                   "parallelism": f"instances sharded over {world} rank(s); NCCL all_gather of 64-B records",
                   "l2": "inputs and workspace larger than L2 (126 MB)"},
        "per_step": {"total_ms": round(total_ms, 3), "build_ms": round(build_ms, 3),
                     "solve_ms": round(solve_ms, 3), "rounds": st["rounds"], "global_relabels": st["global_relabels"],
                     "bfs_levels": st["bfs_levels"], "pushes": st["pushes"], "relabels": st["relabels"],
                     "arcs_scanned": st["arcs_scanned"], "bfs_arcs_scanned": st["bfs_arcs_scanned"],
                     "residual_gteps": round(gteps, 3), "M": st["M"], "flow_total": int(np.sum(flows))},
        "roofline": {"bound": "hbm", "kernel": "k_solve (persistent push-relabel + device GR, 1 launch/step)",
                     "achieved": round(achieved, 2), "peak": hbm, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "algorithmic_bytes_per_launch": int(sb),
                     "launch_ms": round(solve_ms, 3), "traffic": traffic,
                     "build": {"kernels": "A1 construction (st['kernel_launches'] - 4 launches)",
                               "achieved": round(build_achieved, 2), "frac": round(build_achieved / hbm, 4),
                               "algorithmic_bytes": int(bb), "ms": round(build_ms, 3)}},
        "e2e": None if e2e_value is None else {"value": round(e2e_value, 3), "unit": "instances/s" if wl["kind"] == "batch" else "solves/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "pipelined_streams": max(1, args.e2e_streams), "timing": "wall clock between device syncs"},
        "gpu_launches": int(st["kernel_launches"]) * args.steps,
        "clocks": clocks,
        "gen_s": round(gen_s, 2),
    }
    if args.cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(wl, args.cpu_budget_s)
    return out


def run_bipartite(args, rank, world, dev, wl, gen_s):
    """C4 (A9): maximum bipartite matching through wbpr_bipartite_match (network built on
    the device).  value = matchings/s of the whole job (weak scaling: one instance per rank)."""
    import torch
    import torch.distributed as dist
    import paper_2404_00270_b200 as W
    nL, nR = wl["nL"], wl["nR"]
    l_h = torch.from_numpy(wl["l"]).pin_memory()
    r_h = torch.from_numpy(wl["r"]).pin_memory()
    l_d, r_d = l_h.to(dev), r_h.to(dev)
    match_h = torch.empty(nL, dtype=torch.int32).pin_memory()
    opt = dict(layout=args.layout, **WORKLOAD_OPTS.get(args.workload, {}))
    for kv in args.opt:
        k_, v_ = kv.split("=")
        opt[k_] = float(v_) if "." in v_ else int(v_)
    ws = W.Workspace(1 << 20, dev)
    stream = torch.cuda.current_stream(dev)

    def step(host=False):
        if host:   # e2e: inputs H2D from pinned memory and the matching D2H inside the timed region
            l_d.copy_(l_h, non_blocking=True)
            r_d.copy_(r_h, non_blocking=True)
        size, match, st = W.bipartite_match(nL, nR, l_d, r_d, workspace=ws, **opt)
        if host:
            match_h.copy_(match, non_blocking=True)
        return size, match, st

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev.index)
    clk.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sts = []
    ev0.record(stream)
    for _ in range(args.steps):
        size, match, st = step()
        sts.append(st)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    e2e_steps = max(1, min(args.steps, 5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step(host=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    times = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(times[0]), float(times[1])
    if rank != 0:
        return None
    assert size == sts[-1]["flow_value"] == sts[-1]["cut_capacity"]
    hbm, peak_src = peaks()
    solve_ms = float(np.mean([x["solve_ms"] for x in sts]))
    build_ms = float(np.mean([x["build_ms"] for x in sts]))
    total_ms = float(np.mean([x["total_ms"] for x in sts]))
    st = sts[-1]
    sb = solve_bytes(st)
    achieved = sb / (solve_ms / 1e3) / 1e9
    gteps = (st["arcs_scanned"] + st["bfs_arcs_scanned"]) / (solve_ms / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": round(world * args.steps / (ms / 1e3), 3), "unit": "matchings/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "c4", "desc": wl["desc"], "layout": args.layout,
                   "options": {k_: v_ for k_, v_ in opt.items() if k_ != "layout"}, "nL": nL, "nR": nR,
                   "edges": int(wl["l"].shape[0]), "parallelism": f"replicas ({world} rank(s), one instance each)",
                   "l2": "inputs and workspace larger than L2 (126 MB)"},
        "per_step": {"total_ms": round(total_ms, 3), "build_ms": round(build_ms, 3), "solve_ms": round(solve_ms, 3),
                     "rounds": st["rounds"], "global_relabels": st["global_relabels"], "bfs_levels": st["bfs_levels"],
                     "pushes": st["pushes"], "relabels": st["relabels"], "arcs_scanned": st["arcs_scanned"],
                     "bfs_arcs_scanned": st["bfs_arcs_scanned"], "residual_gteps": round(gteps, 3), "M": st["M"],
                     "matching_size": int(size)},
        "roofline": {"bound": "hbm", "kernel": "k_solve (persistent push-relabel + device GR, 1 launch/step)",
                     "achieved": round(achieved, 2), "peak": hbm, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "algorithmic_bytes_per_launch": int(sb),
                     "launch_ms": round(solve_ms, 3), "traffic": None},
        "e2e": {"value": round(world * e2e_steps / (e2e_ms / 1e3), 3), "unit": "matchings/s",
                "h2d_bytes_per_step": int(wl["l"].nbytes + wl["r"].nbytes), "d2h_bytes_per_step": 4 * nL,
                "steps": e2e_steps},
        "gpu_launches": int(st["kernel_launches"]) * args.steps,
        "clocks": clocks,
        "gen_s": round(gen_s, 2),
    }
    if args.cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(wl, args.cpu_budget_s)
    return out


def bipartite_graph(scale=20, l=None, r=None):
    """The C4 matching network (scale 20) or a bounded CPU sample of it: the same recipe at
    2^scale x 2^scale with 2^(scale+4) draws."""
    import synth
    from oracle import matching
    if l is None:
        l, r = synth.bipartite_edges(1 << scale, 1 << scale, 1 << (scale + 4), 1)
    n, src, dst, cap, s, t = matching.network(1 << scale, 1 << scale, l, r)
    return synth.from_edges(n, src, dst, cap, s, t, name=f"c4-network-2^{scale}")


def cpu_baseline(wl, budget_s):
    """The oracle as it stands (oracle/, single thread) on a bounded sample of the workload."""
    import oracle
    if wl["kind"] == "bipartite":
        g = bipartite_graph(20, wl["l"], wl["r"])
        r = oracle.maxflow_graph(g, phase2=False)
        return {"value": round(1.0 / r.seconds, 4), "unit": "matchings/s", "cores": 1, "kind": "oracle",
                "sample": f"the C4 instance itself, one matching: {r.seconds:.2f} s of single-thread oracle "
                          "solve time (ingest excluded)", "cpu": cpu_model(), "nproc": os.cpu_count()}
    parts = wl["parts"] if wl["kind"] == "batch" else [wl["graph"]]
    done, t_sum = 0, 0.0
    for g in parts:
        r = oracle.maxflow_graph(g, phase2=False)
        t_sum += r.seconds
        done += 1
        if t_sum >= budget_s:
            break
    unit = "instances/s" if wl["kind"] == "batch" else "solves/s"
    return {"value": round(done / t_sum, 4), "unit": unit, "cores": 1, "kind": "oracle",
            "sample": f"first {done} of {len(parts)} instance(s) of the workload on this rank, "
                      f"{t_sum:.1f} s of single-thread oracle solve time (ingest excluded)",
            "cpu": cpu_model(), "nproc": os.cpu_count()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle
    wl = make_workload(args.workload, 0, 1)
    if wl["kind"] == "bipartite":
        parts = [bipartite_graph(20, wl["l"], wl["r"])]   # the C4 network itself (~12 s per oracle solve)
    else:
        parts = wl["parts"] if wl["kind"] == "batch" else [wl["graph"]]
    i = 0

    def step():
        nonlocal i
        g = parts[i % len(parts)]
        i += 1
        r = oracle.maxflow_graph(g, phase2=False)
        return r.seconds

    for _ in range(args.warmup):
        step()
    secs = [step() for _ in range(args.steps)]
    t = float(np.sum(secs))
    value = args.steps / t
    unit = {"batch": "instances/s", "bipartite": "matchings/s"}.get(wl["kind"], "solves/s")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if wl["kind"] == "batch" else "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "layout": "oracle arc-pair lists"},
        "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} instance solves of the workload (one per step, cycling)"
                                   + (" - the full C4 network per step" if wl["kind"] == "bipartite" else ""),
                         "cpu": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=["c5", "c1", "c2", "c2r", "c3", "c3h", "c4"])
    ap.add_argument("--layout", default="bcsr", choices=["bcsr", "rcsr"])
    ap.add_argument("--impl", default="wbpr", choices=["wbpr", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--opt", action="append", default=[], help="solver option key=value (wbpr_options field)")
    ap.add_argument("--e2e-streams", type=int, default=2,
                    help="host threads / streams / workspaces issuing the e2e steps (H2D overlaps kernels)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.warmup < 3 and args.impl == "wbpr":
        log("note: warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        out = run_wbpr(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
