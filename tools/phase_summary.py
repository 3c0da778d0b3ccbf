"""Summarise tools/probe.py JSON lines: times, counters and the per-phase-kind breakdown.
usage: python tools/phase_summary.py probe.jsonl"""
import json, sys
NAMES = ["init", "round", "gr_reset", "bfs_td", "compact", "preflow", "gap", "bfs_async", "bfs_bu", "small"]
for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except ValueError:
        continue
    if "phase_ns" not in d:
        continue
    pn, pc = d["phase_ns"], d["phase_count"]
    ph = " ".join(f"{NAMES[i]}:{pn[i] / 1e6:.2f}ms/{pc[i]}" for i in range(len(NAMES)) if pc[i])
    print(f"{d['cfg']:6s} {d['rep']} build {d['build_ms']:.2f} solve {d['solve_ms']:.2f} rounds {d['rounds']} "
          f"grs {d['global_relabels']} lv {d['bfs_levels']} arcs {d['arcs_scanned'] / 1e6:.0f}M "
          f"bfs {d['bfs_arcs_scanned'] / 1e6:.0f}M F {d['flow_value']}")
    print("        ", ph)
