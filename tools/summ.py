import sys, json
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for l in sys.stdin:
    try:
        d = json.loads(l)
    except Exception:
        print(l.rstrip()); continue
    if "rounds" not in d:
        print(tag, d); continue
    ph = d["rounds"] + d["bfs_levels"]
    print(tag, d["cfg"], "F", d["flow_value"], "rounds", d["rounds"], "grs", d["global_relabels"], "levels", d["bfs_levels"],
          "solve_ms", round(d["solve_ms"], 2), "build_ms", round(d["build_ms"], 2), "us/phase", round(1000 * d["solve_ms"] / max(ph, 1), 3),
          "arcs", d["arcs_scanned"], "bfs_arcs", d["bfs_arcs_scanned"], "pushes", d["pushes"], "relabels", d["relabels"], "gaplifts", d["gap_lifts"],
          "t_bar/flush/round_ms", round(d.get("t_barrier_ns", 0) / 1e6, 2), round(d.get("t_flush_ns", 0) / 1e6, 2),
          round(d.get("t_round_ns", 0) / 1e6, 2), flush=True)
