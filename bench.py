#!/usr/bin/env python
"""bench.py — WBPR max-flow hot path on B200 (see DESIGN.md §6 "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c1|c2|c2r|c3|c3h|c4]
                    [--layout bcsr|rcsr] [--impl wbpr|reference] [--dry-run]

One step = one pass of the whole hot path (§8(a) A1-A8, A10: device residual
construction, preflow, push/relabel rounds with device global relabels and
termination, result extraction) over one batch of synthetic input resident in
HBM, through the C-ABI (libwbpr.so).  Default workload (every N): BASELINE.json
configs[4] "C5" — 64 independent R-MAT scale-18 max-flow instances (paper-rule
terminals) partitioned over the N ranks by edge count (one process per GPU),
solved per rank as one disjoint-union batch, results gathered with NCCL
all_gather (at N = 1 too).  value = whole-job instances/s.

The default N = 1 run also carries `per_graph`: the per-graph half of the metric
(solve ms and residual GTEPS) for C3 (R-MAT-22, paper rule and hub20), C4 (2^20 x 2^20
matching) and C2 (1024^2 grid, unit and random capacities) — median / min / max of 5
solves each, roofline fraction, oracle time and bit-exact parity.

Parity gate: after the timed region every instance the run solved is re-solved by the
oracle (oracle/, a process pool over the host cores = the cpu_baseline leg) and the flow
value, cut capacity and canonical cut bitmap are compared element by element.

--gpus N without a torchrun environment re-launches itself under torch.distributed.run
with N ranks.  --impl reference: the CPU oracle (single thread) timed on this host as
the reference arm (rank 0 only).  --dry-run: no GPU; the launcher, the partition by m and
the record gather run over gloo (the CPU test of the N > 1 path).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max-flow solve ms & residual GTEPS per graph (1 B200); batch instances/s at 1/2/4/8"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILES = os.path.join(ROOT, "profiles", "r2")

# Algorithmic bytes per unit of work (restated in DESIGN.md §5)
B_SLOT = 12        # scanned residual slot: col 4 + cf 4 + h[col] 4
B_VERTEX = 32      # processed active vertex: queue 4 + 2 offsets 8 + e 8 + h 4 (+ bookkeeping)
B_PUSH = 52        # mate 4 + two cf RMW 16 + two e RMW 32
B_RELABEL = 4
B_BFS_TD = 16      # top-down in-arc: col 4 + mate 4 + cf[mate] 4 + h[u] 4
B_BFS_BU = 12      # bottom-up out-arc: col 4 + cf 4 + h[col] 4
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
C5_TOTAL = 64


def c5_sizes():
    """(n, m, sha) of the 64 C5 instances (synth/c5_sizes.json, written by tools/c5_sizes.py)."""
    p = os.path.join(ROOT, "synth", "c5_sizes.json")
    try:
        with open(p) as f:
            d = json.load(f)["instances"]
        return [d[str(1000 + i)] for i in range(C5_TOTAL)]
    except Exception:
        return None


def graph_digest(g):
    import hashlib
    h = hashlib.sha256()
    for a in (g.row_off, g.col, g.cap):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(f"{g.s},{g.t}".encode())
    return h.hexdigest()[:32]


def c5_block(rank, world):
    """This rank's contiguous block of C5 instance ids, balanced by edge count m (§8(e))."""
    from paper_2404_00270_b200.batch import partition, partition_weighted
    sz = c5_sizes()
    if sz is None:
        return partition(C5_TOTAL, world, rank), "instance count (synth/c5_sizes.json missing)"
    return partition_weighted([s["m"] for s in sz], world, rank), "edge count m (synth/c5_sizes.json)"


def make_graph(name):
    import synth
    return {"c1": lambda: synth.random_graph(1024, 8192, 1),
            "c2": lambda: synth.grid(1024, 1024, False, 1),
            "c2r": lambda: synth.grid(1024, 1024, True, 1),
            "c3": lambda: synth.rmat(22, 16, 1, "paper"),
            "c3h": lambda: synth.rmat(22, 16, 1, "hub20")}[name]()


def make_workload(name, rank, world):
    """Returns dict(kind, parts|graph, ids, desc) for this rank."""
    import synth
    if name == "c5":
        (lo, hi), how = c5_block(rank, world)
        sz = c5_sizes()
        parts = []
        for i in range(lo, hi):
            g = synth.rmat(18, 16, 1000 + i, "paper")
            if sz is not None:   # the same bytes the size table was written from
                assert g.m == sz[i]["m"] and graph_digest(g) == sz[i]["sha"], f"C5 instance {i} differs from the table"
            parts.append(g)
        counts = [c5_block(r, world)[0][1] - c5_block(r, world)[0][0] for r in range(world)]
        return dict(kind="batch", parts=parts, ids=list(range(lo, hi)), total=C5_TOTAL, partition_by=how,
                    counts=counts,
                    desc="C5: 64 x R-MAT scale 18 (edgefactor 16, U[1,100] caps, 20 paper-rule s/t pairs "
                         "behind super terminals), seeds 1000-1063, partitioned over ranks by m")
    if name == "c4":
        nL = nR = 1 << 20
        l, r = synth.bipartite_edges(nL, nR, 1 << 24, 1)
        return dict(kind="bipartite", nL=nL, nR=nR, l=l, r=r, ids=[rank], total=1,
                    desc="C4: bipartite matching 2^20 x 2^20, 2^24 uniform draws (duplicates collapsed), unit "
                         "capacities via super source/sink (network built on the device, A9)")
    g = make_graph(name)
    return dict(kind="single", graph=g, ids=[rank], total=1, desc=g.name)


def bipartite_graph(scale=20, l=None, r=None):
    """The C4 matching network (scale 20) as a max-flow instance (for the oracle)."""
    import synth
    from oracle import matching
    if l is None:
        l, r = synth.bipartite_edges(1 << scale, 1 << scale, 1 << (scale + 4), 1)
    n, src, dst, cap, s, t = matching.network(1 << scale, 1 << scale, l, r)
    return synth.from_edges(n, src, dst, cap, s, t, name=f"c4-network-2^{scale}")


# ---------------------------------------------------------------------------- oracle pool
# The cpu_baseline leg: the oracle (oracle/, FIFO push-relabel + gap, single-threaded C with
# no global state) run over the host cores by a pool of threads - ctypes releases the GIL for
# the duration of each C call, so every worker solves on its own core - over the very instance
# arrays the GPU solved.  Used for the parity gate and timed as the all-core oracle throughput
# (SURVEY §8(d) "Oracle timing").
_POOL_GRAPHS = {}


def _oracle_task(key):
    import oracle
    r = oracle.maxflow_graph(_POOL_GRAPHS[key], phase2=False)
    return key, r.flow, r.cut_capacity, r.bitmap_words(), r.seconds


class OraclePool:
    def __init__(self, graphs: dict, workers: int):
        import concurrent.futures as cf
        import oracle
        oracle.build()
        _POOL_GRAPHS.clear()
        _POOL_GRAPHS.update(graphs)
        self.workers = max(1, min(workers, len(graphs) or 1))
        self.pool = cf.ThreadPoolExecutor(self.workers)

    def run(self, keys):
        t0 = time.perf_counter()
        res = {k: (f, c, b, s) for k, f, c, b, s in self.pool.map(_oracle_task, keys)}
        return res, time.perf_counter() - t0

    def close(self):
        self.pool.shutdown()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


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
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def solve_bytes(st):
    """Algorithmic bytes moved by one launch of the persistent solve kernel, from that
    launch's own counters (§5): top-down BFS arcs at 16 B, bottom-up ones at 12 B."""
    bu = st.get("bfs_arcs_bottom_up", 0)
    td = st["bfs_arcs_scanned"] - bu
    return (B_SLOT * st["arcs_scanned"] + B_VERTEX * st["avq_total"] + B_PUSH * st["pushes"] +
            B_RELABEL * st["relabels"] + B_BFS_TD * td + B_BFS_BU * bu +
            B_GR_VERTEX * st["n"] * st["global_relabels"] + B_CAND * st["compaction_candidates"])


def build_bytes(st):
    """Algorithmic bytes of construction A1 (BCSR merge build): read the input CSR (8 B per
    edge + 8 B per row), write+read the 8-B out-keys and the 4-B in-list entries once, write
    16 B per output slot (arc 8 + mate 4 + cap0 4)."""
    m, n, M = st["m"], st["n"], st["M"]
    return 8 * m + 8 * n + 2 * 8 * m + 2 * 4 * m + 16 * M


def roofline_of(sts, hbm):
    """Achieved GB/s of the solve kernel over several launches: sum of each launch's own
    algorithmic bytes over the sum of its own CUDA-event times (same run, same launch)."""
    b = [solve_bytes(s) for s in sts]
    t = [s["solve_ms"] for s in sts]
    fr = [bi / (ti / 1e3) / 1e9 / hbm for bi, ti in zip(b, t) if ti > 0]
    ach = sum(b) / (sum(t) / 1e3) / 1e9
    td = sum(s["bfs_arcs_scanned"] - s.get("bfs_arcs_bottom_up", 0) for s in sts)
    bu = sum(s.get("bfs_arcs_bottom_up", 0) for s in sts)
    return {"achieved": round(ach, 2), "frac": round(ach / hbm, 4),
            "frac_per_launch": {"median": round(float(np.median(fr)), 4), "min": round(min(fr), 4),
                                "max": round(max(fr), 4)},
            "algorithmic_bytes_per_launch": int(sum(b) / len(b)), "launch_ms": round(sum(t) / len(t), 3),
            "launches": len(sts),
            "bytes_by_unit": {"slots": B_SLOT, "vertex": B_VERTEX, "push": B_PUSH, "relabel": B_RELABEL,
                              "bfs_arc_top_down": B_BFS_TD, "bfs_arc_bottom_up": B_BFS_BU,
                              "gr_vertex": B_GR_VERTEX, "candidate": B_CAND},
            "bfs_arcs_top_down_per_launch": int(td / len(sts)), "bfs_arcs_bottom_up_per_launch": int(bu / len(sts))}


def traffic_of(workload, layout):
    """DRAM bytes of one solve launch from ncu, captured in the SAME launch as its own
    algorithmic byte count (tools/traffic_run.py -> profiles/r2/traffic_<workload>_<layout>.json)."""
    p = os.path.join(PROFILES, f"traffic_{workload}_{layout}.json")
    if not os.path.exists(p):
        return None, None
    try:
        d = json.load(open(p))
        return d["dram_bytes_per_launch"], {k: d[k] for k in ("dram_bytes_per_launch", "algorithmic_bytes_per_launch",
                                                               "ratio", "l2_hit_pct", "warp_efficiency",
                                                               "launches", "source") if k in d}
    except Exception:
        return None, None


def stat3(xs, nd=3):
    xs = [float(x) for x in xs]
    return {"median": round(float(np.median(xs)), nd), "min": round(min(xs), nd), "max": round(max(xs), nd)}


def latency_floor(sts, ns_phase):
    """Barrier-latency floor of a solve: grid-synchronous phases x the measured cost of an
    EMPTY phase (wbpr_barrier_cost); small-frontier spans run on block barriers (excluded)."""
    if not ns_phase:
        return None
    ph = [sum(s["phase_count"][:9]) for s in sts]
    small = [s["phase_count"][9] for s in sts]
    fl = [p * ns_phase / 1e6 for p in ph]
    names = ["none", "round", "gr_reset", "bfs_top_down", "compact", "preflow", "gap_lift", "async_bfs",
             "bfs_bottom_up", "small_mode"]
    by_kind = {nm: {"ms": round(float(np.median([s["phase_ns"][i] for s in sts]) / 1e6), 3),
                    "phases": int(np.median([s["phase_count"][i] for s in sts]))}
               for i, nm in enumerate(names) if any(s["phase_count"][i] for s in sts)}
    return {"grid_phases_per_solve": int(np.median(ph)), "small_mode_phases_per_solve": int(np.median(small)),
            "ns_per_empty_phase": round(ns_phase, 1), "floor_ms": round(float(np.median(fl)), 3),
            "floor_share_of_solve": round(float(np.median([f / s["solve_ms"] for f, s in zip(fl, sts)])), 4),
            "phase_time_by_kind": by_kind}


# ---------------------------------------------------------------------------- device helpers
def flush_l2(dev, buf=[]):
    import torch
    if not buf:
        buf.append(torch.empty(256 << 20, dtype=torch.uint8, device=dev))
    buf[0].fill_(1)


# per-graph sub-lines with their own solver options, and sub-lines whose instance another
# sub-line already hands to the oracle pool
SUBLINE_OPTS = {"c3h_pm0": {"push_mode": 0}}
ORACLE_ALIAS = {"c3h_pm0": "c3h"}


def parse_opts(args, workload):
    opt = dict(layout=args.layout, **WORKLOAD_OPTS.get(workload, {}))
    for kv in args.opt:
        k_, v_ = kv.split("=")
        opt[k_] = float(v_) if "." in v_ else int(v_)
    return opt


def graph_line(name, g, dev, layout, reps=5, warmup=2, opt=None, ns_phase=None):
    """Per-graph sub-line: `reps` device-resident solves (each preceded by an L2 flush),
    median / min / max of the library's own CUDA-event windows, roofline from each solve's
    own counters; returns (line, gpu result for the parity gate)."""
    import torch
    import paper_2404_00270_b200 as W
    opt = dict(opt or {})
    ro, col, cap = (torch.from_numpy(a).to(dev) for a in (g.row_off, g.col, g.cap))
    ws = W.Workspace(W.workspace_size(g.n, g.m, 1, W.options(layout)), dev)
    sts = []
    for i in range(warmup + reps):
        flush_l2(dev)
        torch.cuda.synchronize(dev)
        F, bm, st = W.maxflow(ro, col, cap, g.s, g.t, layout=layout, workspace=ws, device=dev, **opt)
        if i >= warmup:
            sts.append(st)
    words = bm.cpu().numpy().view(np.uint32).copy()
    hbm, _ = peaks()
    gteps = [(s["arcs_scanned"] + s["bfs_arcs_scanned"]) / (s["solve_ms"] / 1e3) / 1e9 for s in sts]
    med = sorted(sts, key=lambda s: s["total_ms"])[len(sts) // 2]
    line = {"workload": name, "desc": g.name, "layout": layout, "options": opt, "n": g.n, "m": g.m, "M": med["M"],
            "reps": reps,
            "total_ms": stat3([s["total_ms"] for s in sts]), "build_ms": stat3([s["build_ms"] for s in sts]),
            "solve_ms": stat3([s["solve_ms"] for s in sts]), "residual_gteps": stat3(gteps),
            "m_per_total_ms_gteps": round(g.m / (med["total_ms"] / 1e3) / 1e9, 3),
            "counters_median_run": {k: med[k] for k in ("rounds", "global_relabels", "bfs_levels", "pushes", "relabels",
                                                        "arcs_scanned", "bfs_arcs_scanned", "bfs_arcs_bottom_up")},
            "roofline": dict(bound="hbm", kernel="k_solve", peak=hbm, unit="GB/s", **roofline_of(sts, hbm)),
            "latency_floor": latency_floor(sts, ns_phase),
            "flow": int(F), "cut_capacity": int(med["cut_capacity"])}
    tr, tr_cap = traffic_of(name, layout)
    line["roofline"]["traffic"] = tr
    line["roofline"]["traffic_same_capture"] = tr_cap
    del ws, ro, col, cap
    torch.cuda.empty_cache()
    return line, (int(F), int(med["cut_capacity"]), words)


def bipartite_line(wl, dev, layout, reps=5, warmup=2, ns_phase=None):
    import torch
    import paper_2404_00270_b200 as W
    nL, nR = wl["nL"], wl["nR"]
    l_d = torch.from_numpy(wl["l"]).to(dev)
    r_d = torch.from_numpy(wl["r"]).to(dev)
    ws = W.Workspace(1 << 20, dev)
    sts = []
    for i in range(warmup + reps):
        flush_l2(dev)
        torch.cuda.synchronize(dev)
        size, match, st = W.bipartite_match(nL, nR, l_d, r_d, layout=layout, workspace=ws)
        if i >= warmup:
            sts.append(st)
    hbm, _ = peaks()
    gteps = [(s["arcs_scanned"] + s["bfs_arcs_scanned"]) / (s["solve_ms"] / 1e3) / 1e9 for s in sts]
    med = sorted(sts, key=lambda s: s["total_ms"])[len(sts) // 2]
    line = {"workload": "c4", "desc": wl["desc"], "layout": layout, "nL": nL, "nR": nR, "edges": int(wl["l"].shape[0]),
            "M": med["M"], "reps": reps, "total_ms": stat3([s["total_ms"] for s in sts]),
            "build_ms": stat3([s["build_ms"] for s in sts]), "solve_ms": stat3([s["solve_ms"] for s in sts]),
            "residual_gteps": stat3(gteps),
            "counters_median_run": {k: med[k] for k in ("rounds", "global_relabels", "bfs_levels", "pushes", "relabels",
                                                        "arcs_scanned", "bfs_arcs_scanned", "bfs_arcs_bottom_up")},
            "roofline": dict(bound="hbm", kernel="k_solve", peak=hbm, unit="GB/s", **roofline_of(sts, hbm)),
            "latency_floor": latency_floor(sts, ns_phase),
            "matching_size": int(size)}
    tr, tr_cap = traffic_of("c4", layout)
    line["roofline"]["traffic"] = tr
    line["roofline"]["traffic_same_capture"] = tr_cap
    m_host = match.cpu().numpy().copy()
    del ws, l_d, r_d
    torch.cuda.empty_cache()
    return line, (int(size), int(med["cut_capacity"]), m_host)


# ---------------------------------------------------------------------------- wbpr arm
def run_wbpr(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2404_00270_b200 as W

    t0 = time.time()
    wl = make_workload(args.workload, rank, world)
    extra = {}   # per-graph sub-line instances (N = 1 default run)
    if args.per_graph and world == 1 and args.workload == "c5":
        import synth
        g3 = synth.rmat(22, 16, 1, "paper")
        g3h = synth.rmat(22, 16, 1, "hub20")
        # c3h_pm0: the same C3-hub20 instance under the paper's single push per active vertex
        # (Alg. 2, push_mode 0) - the cost of the warp-parallel discharge deviation at full size
        extra = {"c3": g3, "c3h": g3h, "c3h_pm0": g3h, "c2": make_graph("c2"), "c2r": make_graph("c2r")}
        l4, r4 = synth.bipartite_edges(1 << 20, 1 << 20, 1 << 24, 1)
        extra["c4"] = dict(kind="bipartite", nL=1 << 20, nR=1 << 20, l=l4, r=r4,
                           desc="C4: bipartite matching 2^20 x 2^20, 2^24 uniform draws, unit capacities")
    gen_s = time.time() - t0
    # ---- the oracle pool (cpu_baseline leg + parity gate), run after all device timing
    pool = None
    if args.cpu_baseline:
        graphs = {}
        if wl["kind"] == "batch":
            for i, g in zip(wl["ids"], wl["parts"]):
                graphs[("c5", i)] = g
        elif wl["kind"] == "single":
            graphs[(args.workload, 0)] = wl["graph"]
        else:
            graphs[("c4", 0)] = bipartite_graph(20, wl["l"], wl["r"])
        for k_, g in extra.items():
            if k_ in ORACLE_ALIAS:
                continue   # same instance as another sub-line: one oracle run serves both
            graphs[(k_, 0)] = bipartite_graph(20, g["l"], g["r"]) if isinstance(g, dict) else g
        pool = OraclePool(graphs, max(1, host_cores() // world))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    init_group("nccl", rank, world, dev)
    if wl["kind"] == "bipartite":
        out = run_bipartite_main(args, rank, world, dev, wl, gen_s, pool)
        if pool:
            pool.close()
        return out
    if wl["kind"] == "batch":
        import synth
        B = synth.disjoint_union(wl["parts"])
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
    opt = parse_opts(args, args.workload)
    ws = W.Workspace(W.workspace_size(G.n, G.m, k, W.options(args.layout)), dev)
    bitmap_d = torch.empty((G.n + 31) // 32, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    from paper_2404_00270_b200.batch import gather_records_async, make_records, order_records
    gathered = None
    dumped = []
    counts = wl.get("counts", [1] * world)
    rec_h = torch.empty((len(wl["ids"]), 8), dtype=torch.int64).pin_memory()
    rec_d = torch.empty((len(wl["ids"]), 8), dtype=torch.int64, device=dev)

    def step():
        flows, cuts, _, st = W.maxflow_batch(ro_d, col_d, cap_d, vbase, s, t, workspace=ws, bitmap=bitmap_d,
                                             device=dev, **opt)
        # 64-B result record per instance (id, status, F, cut, rounds, GRs, pushes, relabels),
        # gathered over ranks: the only collective (NCCL all_gather_into_tensor, every N; no
        # host synchronisation inside the step - the records are checked after the timed loop)
        nonlocal gathered
        rec_h.numpy()[:] = make_records(wl["ids"], flows, cuts, st)
        rec_d.copy_(rec_h, non_blocking=True)
        gathered = gather_records_async(rec_d, counts, world)
        if args.dump_steps:
            dumped.append(dict(solve_bytes=solve_bytes(st), **{k_: v_ for k_, v_ in st.items()
                                                               if not isinstance(v_, list)}))
        return st, flows, cuts

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local_rank)
    clk.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    sts = []
    dist.barrier()
    torch.cuda.synchronize(dev)
    evs[0].record(stream)
    for i in range(args.steps):
        st, flows, cuts = step()
        evs[i + 1].record(stream)
        sts.append(st)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = clk.stop()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms = evs[0].elapsed_time(evs[-1])
    bm_gpu = bitmap_d.cpu().numpy().view(np.uint32).copy()
    flows_gpu, cuts_gpu = np.asarray(flows).copy(), np.asarray(cuts).copy()
    if args.dump_steps:
        with open(f"{args.dump_steps}.rank{rank}", "w") as f:
            json.dump(dumped, f)
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
    dist.barrier()
    t0 = time.perf_counter()
    if len(pipes) == 1:
        host_steps(pipes[0], e2e_steps)
    elif pipes:
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
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(times[0]), float(times[1])
    total_units = wl["total"] if wl["kind"] == "batch" else world
    value = total_units * args.steps / (ms / 1e3)
    e2e_value = total_units * e2e_steps / (e2e_ms / 1e3) if args.e2e_streams > 0 else None
    del ws
    torch.cuda.empty_cache()
    # ---- barrier-latency floor (an empty grid phase of the persistent kernel)
    try:
        ns_phase = W.barrier_cost(0, 4000, dev)
    except Exception as ex:   # measurement helper only
        log("barrier probe failed:", ex)
        ns_phase = None
    # ---- per-graph sub-lines (device work; N = 1 default run)
    per_graph, gpu_extra = {}, {}
    for name, g in extra.items():
        if isinstance(g, dict):
            per_graph[name], gpu_extra[name] = bipartite_line(g, dev, args.layout, ns_phase=ns_phase)
        else:
            slow = name in ("c2r", "c3h_pm0")
            per_graph[name], gpu_extra[name] = graph_line(name, g, dev, args.layout, reps=3 if slow else 5,
                                                          warmup=1 if slow else 2, ns_phase=ns_phase,
                                                          opt=SUBLINE_OPTS.get(name))
    # ---- parity gate + cpu_baseline leg (after all device timing)
    parity, cpu = None, None
    if pool is not None:
        # first this rank's own workload alone (its wall time is the all-core oracle rate),
        # then the per-graph instances
        batch_keys = [k_ for k_ in _POOL_GRAPHS if k_[0] == args.workload]
        res, wall = pool.run(batch_keys)
        if per_graph:
            res2, _ = pool.run([(name, 0) for name in per_graph if name not in ORACLE_ALIAS])
            res.update(res2)
        pool.close()
        mism = []
        checked = 0
        if wl["kind"] == "batch":
            words = bm_gpu
            for j, i in enumerate(wl["ids"]):
                f, c, bw, _ = res[("c5", i)]
                lo_, hi_ = int(vbase[j]), int(vbase[j + 1])
                ok = flows_gpu[j] == f and cuts_gpu[j] == c and slice_equal(words, lo_, hi_, bw)
                checked += 1
                if not ok:
                    mism.append(i)
        elif wl["kind"] == "single":
            f, c, bw, _ = res[(args.workload, 0)]
            checked = 1
            if not (int(flows_gpu[0]) == f and int(cuts_gpu[0]) == c and np.array_equal(bm_gpu, bw)):
                mism.append(0)
        mm = torch.tensor([len(mism), checked], dtype=torch.int64, device=dev)
        dist.all_reduce(mm)
        parity = {"instances": int(mm[1]), "mismatches": int(mm[0]), "compared": "flow, cut capacity, cut bitmap "
                  "(bit-exact, element by element)", "against": "oracle/ (FIFO push-relabel + gap, C)",
                  "mismatched_ids_this_rank": mism}
        for name in per_graph:
            f, c, bw, osec = res[(ORACLE_ALIAS.get(name, name), 0)]
            gf, gc, gw = gpu_extra[name]
            if name == "c4":
                from oracle import matching
                ok_valid = True
                try:
                    matching.check_matching(extra["c4"]["nL"], extra["c4"]["nR"], extra["c4"]["l"], extra["c4"]["r"],
                                            gw, gf)
                except AssertionError:
                    ok_valid = False
                per_graph[name]["parity"] = {"size_equals_oracle_flow": gf == f, "matching_valid": ok_valid}
                bad = not (gf == f and ok_valid)
            else:
                eq = {"flow": gf == f, "cut_capacity": gc == c, "bitmap": bool(np.array_equal(gw, bw))}
                per_graph[name]["parity"] = eq
                bad = not all(eq.values())
            per_graph[name]["oracle"] = {"seconds_1_core": round(osec, 3), "flow": f, "cores": 1}
            per_graph[name]["speedup_vs_oracle_total"] = round(osec / (per_graph[name]["total_ms"]["median"] / 1e3), 1)
            if bad:
                parity["mismatches"] += 1
            parity["instances"] += 1
        secs = [res[k_][3] for k_ in batch_keys]
        nb_ = len(batch_keys)
        if rank == 0 and world == 1:   # (the contract's cpu_baseline is N = 1 only; the parity gate runs at every N)
            cpu = {"value": round(nb_ / wall, 4), "unit": "instances/s" if wl["kind"] == "batch" else "solves/s",
                   "cores": min(pool.workers, nb_), "kind": "oracle",
                   "sample": f"every instance of this rank's workload ({nb_}), oracle solve on a process pool of "
                             f"{min(pool.workers, nb_)} worker(s) over the host cores, wall clock of the pool "
                             f"(instances already in memory; ingest inside each solve call)",
                   "single_core": {"value": round(nb_ / sum(secs), 4), "seconds_per_instance": round(sum(secs) / nb_, 4),
                                   "cores": 1, "timing": "oracle solve only (ingest excluded)"},
                   "cpu": cpu_model(), "nproc": os.cpu_count(), "pool_wall_s": round(wall, 2)}
    if rank != 0:
        return None
    # certificate of every gathered record: F == cut capacity
    g = order_records(gathered, wl["total"] if wl["kind"] == "batch" else world).cpu().numpy()
    assert np.all(g[:, 2] == g[:, 3]), "certificate failed in gathered records"
    hbm, peak_src = peaks()
    st = sts[-1]
    roof = roofline_of(sts, hbm)
    traffic, traffic_cap = traffic_of(args.workload, args.layout)
    bsum = sum(build_bytes(x) for x in sts)
    btime = sum(x["build_ms"] for x in sts)
    build_achieved = bsum / (btime / 1e3) / 1e9
    gteps = [(x["arcs_scanned"] + x["bfs_arcs_scanned"]) / (x["solve_ms"] / 1e3) / 1e9 for x in sts]
    h2d = int(G.row_off.nbytes + G.col.nbytes + G.cap.nbytes)
    d2h = int((G.n + 31) // 32 * 4 + 16 * k)
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
                   "partition": wl.get("partition_by", "one instance per rank"),
                   "parallelism": f"instances sharded over {world} rank(s) (no data-path collective); "
                                  f"NCCL all_gather of 64-B result records",
                   "l2": "inputs and workspace larger than L2 (126 MB): no flush between steps"},
        "per_step_ms": stat3(step_ms),
        "per_step": {"total_ms": stat3([x["total_ms"] for x in sts]), "build_ms": stat3([x["build_ms"] for x in sts]),
                     "solve_ms": stat3([x["solve_ms"] for x in sts]), "rounds": st["rounds"],
                     "global_relabels": st["global_relabels"], "bfs_levels": st["bfs_levels"], "pushes": st["pushes"],
                     "relabels": st["relabels"], "arcs_scanned": st["arcs_scanned"],
                     "bfs_arcs_scanned": st["bfs_arcs_scanned"], "bfs_arcs_bottom_up": st["bfs_arcs_bottom_up"],
                     "residual_gteps": stat3(gteps), "M": st["M"], "flow_total": int(np.sum(flows_gpu))},
        "roofline": {"bound": "hbm", "kernel": "k_solve (persistent push-relabel + device GR, 1 launch/step)",
                     "achieved": roof["achieved"], "peak": hbm, "peak_source": peak_src, "unit": "GB/s",
                     "frac": roof["frac"], "traffic": traffic, "traffic_same_capture": traffic_cap,
                     "detail": roof,
                     "build": {"kernels": "A1 construction (all launches before k_solve)",
                               "achieved": round(build_achieved, 2), "frac": round(build_achieved / hbm, 4),
                               "algorithmic_bytes": int(bsum / len(sts)), "ms": round(btime / len(sts), 3)}},
        "latency_floor": latency_floor(sts, ns_phase),
        "e2e": None if e2e_value is None else {
            "value": round(e2e_value, 3), "unit": "instances/s" if wl["kind"] == "batch" else "solves/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
            "pipelined_streams": max(1, args.e2e_streams), "timing": "wall clock between device syncs"},
        "gpu_launches": int(sum(x["kernel_launches"] for x in sts)),
        "clocks": clocks,
        "gen_s": round(gen_s, 2),
    }
    if parity is not None:
        out["parity"] = parity
    if per_graph:
        out["per_graph"] = per_graph
    if cpu is not None:
        out["cpu_baseline"] = cpu
    return out


def slice_equal(words, lo, hi, ref_words):
    """Bits [lo, hi) of the union bitmap `words` == the instance's own bitmap `ref_words`."""
    bits = np.unpackbits(np.asarray(words, np.uint32).view(np.uint8), bitorder="little")[lo:hi]
    ref = np.unpackbits(np.asarray(ref_words, np.uint32).view(np.uint8), bitorder="little")
    return np.array_equal(bits, ref[:hi - lo]) and not ref[hi - lo:].any()


def run_bipartite_main(args, rank, world, dev, wl, gen_s, pool):
    """C4 (A9) as the main line: maximum bipartite matching through wbpr_bipartite_match (network
    built on the device).  value = matchings/s of the whole job (weak scaling: one per rank)."""
    import torch
    import torch.distributed as dist
    import paper_2404_00270_b200 as W
    nL, nR = wl["nL"], wl["nR"]
    l_h = torch.from_numpy(wl["l"]).pin_memory()
    r_h = torch.from_numpy(wl["r"]).pin_memory()
    l_d, r_d = l_h.to(dev), r_h.to(dev)
    match_h = torch.empty(nL, dtype=torch.int32).pin_memory()
    opt = parse_opts(args, args.workload)
    ws = W.Workspace(1 << 20, dev)
    stream = torch.cuda.current_stream(dev)

    def step(host=False):
        if host:   # e2e: inputs H2D from pinned memory and the matching D2H inside the timed region
            l_d.copy_(l_h, non_blocking=True)
            r_d.copy_(r_h, non_blocking=True)
        size, match, st = W.bipartite_match(nL, nR, l_d, r_d, workspace=ws, **opt)
        if host:
            match_h.copy_(match, non_blocking=True)
        elif args.dump_steps:
            dumped.append(dict(solve_bytes=solve_bytes(st), **{k_: v_ for k_, v_ in st.items()
                                                               if not isinstance(v_, list)}))
        return size, match, st

    dumped = []

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(dev.index)
    clk.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    sts = []
    evs[0].record(stream)
    for i in range(args.steps):
        size, match, st = step()
        evs[i + 1].record(stream)
        sts.append(st)
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = clk.stop()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    m_gpu = match.cpu().numpy().copy()
    if args.dump_steps:
        with open(f"{args.dump_steps}.rank{rank}", "w") as f:
            json.dump(dumped, f)
    e2e_steps = max(1, min(args.steps, 5)) if args.e2e_streams > 0 else 0   # 0: profiler runs (no e2e leg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step(host=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1) if e2e_steps else float("nan")
    times = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(times, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(times[0]), float(times[1])
    parity, cpu = None, None
    if pool is not None:
        res, wall = pool.run([("c4", 0)])
        pool.close()
        f, c, _, osec = res[("c4", 0)]
        from oracle import matching
        ok = True
        try:
            matching.check_matching(nL, nR, wl["l"], wl["r"], m_gpu, int(size))
        except AssertionError:
            ok = False
        parity = {"instances": 1, "mismatches": 0 if (ok and int(size) == f) else 1,
                  "compared": "matching size == oracle max-flow value; matching validity (pairs are input edges, "
                              "each vertex at most once)"}
        cpu = {"value": round(1.0 / osec, 4), "unit": "matchings/s", "cores": 1, "kind": "oracle",
               "sample": f"the C4 network itself, one matching: {osec:.2f} s of single-thread oracle solve time "
                         "(ingest excluded)", "cpu": cpu_model(), "nproc": os.cpu_count()}
    if rank != 0:
        return None
    assert size == sts[-1]["flow_value"] == sts[-1]["cut_capacity"]
    hbm, peak_src = peaks()
    roof = roofline_of(sts, hbm)
    traffic, traffic_cap = traffic_of("c4", args.layout)
    gteps = [(x["arcs_scanned"] + x["bfs_arcs_scanned"]) / (x["solve_ms"] / 1e3) / 1e9 for x in sts]
    st = sts[-1]
    out = {
        "metric": METRIC, "value": round(world * args.steps / (ms / 1e3), 3), "unit": "matchings/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "c4", "desc": wl["desc"], "layout": args.layout,
                   "options": {k_: v_ for k_, v_ in opt.items() if k_ != "layout"}, "nL": nL, "nR": nR,
                   "edges": int(wl["l"].shape[0]), "parallelism": f"replicas ({world} rank(s), one instance each)",
                   "l2": "inputs and workspace larger than L2 (126 MB)"},
        "per_step_ms": stat3(step_ms),
        "per_step": {"total_ms": stat3([x["total_ms"] for x in sts]), "build_ms": stat3([x["build_ms"] for x in sts]),
                     "solve_ms": stat3([x["solve_ms"] for x in sts]), "rounds": st["rounds"],
                     "global_relabels": st["global_relabels"], "bfs_levels": st["bfs_levels"],
                     "pushes": st["pushes"], "relabels": st["relabels"], "arcs_scanned": st["arcs_scanned"],
                     "bfs_arcs_scanned": st["bfs_arcs_scanned"], "bfs_arcs_bottom_up": st["bfs_arcs_bottom_up"],
                     "residual_gteps": stat3(gteps), "M": st["M"], "matching_size": int(size)},
        "roofline": {"bound": "hbm", "kernel": "k_solve (persistent push-relabel + device GR, 1 launch/step)",
                     "achieved": roof["achieved"], "peak": hbm, "peak_source": peak_src, "unit": "GB/s",
                     "frac": roof["frac"], "traffic": traffic, "traffic_same_capture": traffic_cap, "detail": roof},
        "e2e": {"value": round(world * e2e_steps / (e2e_ms / 1e3), 3) if e2e_steps else None, "unit": "matchings/s",
                "h2d_bytes_per_step": int(wl["l"].nbytes + wl["r"].nbytes), "d2h_bytes_per_step": 4 * nL,
                "steps": e2e_steps},
        "gpu_launches": int(sum(x["kernel_launches"] for x in sts)),
        "clocks": clocks,
        "gen_s": round(gen_s, 2),
    }
    if parity is not None:
        out["parity"] = parity
    if cpu is not None:
        out["cpu_baseline"] = cpu
    return out


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle
    wl = make_workload(args.workload, 0, 1) if args.workload != "c5" else None
    if args.workload == "c5":   # the first instances of the workload, generated as needed
        import synth
        parts = [synth.rmat(18, 16, 1000 + i, "paper") for i in range(min(C5_TOTAL, max(1, args.steps)))]
        desc = ("C5: 64 x R-MAT scale 18 (edgefactor 16, U[1,100] caps, 20 paper-rule s/t pairs behind super "
                "terminals), seeds 1000-1063")
        kind = "batch"
    elif wl["kind"] == "bipartite":
        parts = [bipartite_graph(20, wl["l"], wl["r"])]   # the C4 network itself (~6-12 s per oracle solve)
        desc, kind = wl["desc"], "bipartite"
    else:
        parts = [wl["graph"]]
        desc, kind = wl["desc"], "single"
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
    unit = {"batch": "instances/s", "bipartite": "matchings/s"}.get(kind, "solves/s")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3),
        "higher_is_better": True, "scaling": "strong" if kind == "batch" else "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": desc, "layout": "oracle arc-pair lists"},
        "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} instance solves of the workload (one per step, cycling)"
                                   + (" - the full C4 network per step" if kind == "bipartite" else ""),
                         "cpu": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------------------- launcher / process group
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """`--gpus N` outside a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    log("launching:", " ".join(cmd))
    return subprocess.run(cmd).returncode


def init_group(backend, rank, world, dev=None):
    """One process group at every world size (NCCL accepts world 1), so the record gather is a
    real collective at N = 1 as well."""
    import torch.distributed as dist
    if dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    kw = {"device_id": dev} if (backend == "nccl" and dev is not None) else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)


def run_dry(args, rank, world):
    """No GPU: the launcher, the partition by m and the record gather over gloo (CPU test of the
    N > 1 path).  Prints a line marked dry_run; no solve runs and nothing is measured."""
    import torch
    from paper_2404_00270_b200.batch import gather_records, make_records
    init_group("gloo", rank, world)
    (lo, hi), how = c5_block(rank, world)
    ids = list(range(lo, hi))
    rec = torch.from_numpy(make_records(ids, [-1] * len(ids), [-1] * len(ids)))
    allrec = gather_records(rec, C5_TOTAL, world)
    import torch.distributed as dist
    blocks = [None] * world
    dist.all_gather_object(blocks, [lo, hi])
    if rank != 0:
        return None
    sz = c5_sizes()
    ms = [sum(sz[i]["m"] for i in range(a, b)) for a, b in blocks] if sz else None
    return {"dry_run": True, "n_gpus": world, "backend": "gloo", "workload": "c5", "partition": blocks,
            "partition_by": how, "m_per_rank": ms, "records_gathered": int(allrec.shape[0]),
            "ids_ok": bool((allrec[:, 0] == torch.arange(C5_TOTAL)).all())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=["c5", "c1", "c2", "c2r", "c3", "c3h", "c4"])
    ap.add_argument("--layout", default="bcsr", choices=["bcsr", "rcsr"])
    ap.add_argument("--impl", default="wbpr", choices=["wbpr", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false",
                    help="skip the oracle pool (parity gate + cpu_baseline)")
    ap.add_argument("--no-per-graph", dest="per_graph", action="store_false",
                    help="skip the C3/C3h/C4/C2/C2r sub-lines of the default run")
    ap.add_argument("--opt", action="append", default=[], help="solver option key=value (wbpr_options field)")
    ap.add_argument("--e2e-streams", type=int, default=2,
                    help="host threads / streams / workspaces issuing the e2e steps (H2D overlaps kernels)")
    ap.add_argument("--dump-steps", default="", help="write every step's counters (warm-up included) to FILE.rankR")
    ap.add_argument("--dry-run", action="store_true", help="no GPU: launcher + partition + gather over gloo")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(env_world or 1)
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.warmup < 3 and args.impl == "wbpr" and not args.dry_run:
        log("note: warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.dry_run:
        out = run_dry(args, rank, world)
    elif args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_wbpr(args, rank, world, local_rank)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
