#!/bin/bash
# Default bench line (C5 + per-graph sub-lines + parity gate) and the C5 launch list.
O=gpurun_out/${TAG:-b}
mkdir -p $O
timeout 900 python bench.py ${BARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
tail -1 $O/bench.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['per_step']
print('value',d['value'],'build',p['build_ms']['median'],'solve',p['solve_ms']['median'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],'parity',d.get('parity',{}).get('mismatches'))
for k,v in d.get('per_graph',{}).items(): print(k, v['total_ms']['median'], v['build_ms']['median'], v['solve_ms']['median'], v['roofline']['frac'], v['parity'])"
if [ -z "$NOLAUNCH" ]; then
  timeout 600 bash tools/build_profile.sh > /dev/null 2>&1; cp gpurun_out/bp/launches_c5_summary.txt $O/ 2>/dev/null
  head -16 $O/launches_c5_summary.txt
fi
