for b in 0 148 64; do timeout 120 python tools/probe.py path20000 --reps 2 --blocks $b | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['cfg'],'blocks',d['grid_blocks'],'rounds',d['rounds'],'levels',d['bfs_levels'],'solve_ms',round(d['solve_ms'],2),'us/phase',round(1000*d['solve_ms']/(d['rounds']+d['bfs_levels']),3))"; done
for beta in 0.02 0.1 0.5 2; do timeout 200 python tools/probe.py c4 g256r --reps 1 --beta $beta | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['cfg'],'beta',$beta,'rounds',d['rounds'],'grs',d['global_relabels'],'levels',d['bfs_levels'],'solve_ms',round(d['solve_ms'],1),'arcs',d['arcs_scanned'],'bfsarcs',d['bfs_arcs_scanned'])"; done
