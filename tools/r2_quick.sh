#!/bin/bash
# Quick GPU check after a build change: focused parity tests, a short C5 bench, the C5 launch list.
O=gpurun_out/${TAG:-q}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiny.py tests/test_gpu_state.py -m gpu -x -q -p no:cacheprovider ${PYK:+-k "$PYK"} > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
tail -2 $O/tests.txt
if [ -n "$FULL" ]; then
  timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider > $O/tests_full.txt 2>&1; echo "rc=$?" >> $O/tests_full.txt
  tail -2 $O/tests_full.txt
fi
timeout 600 python bench.py --workload ${WL:-c5} --steps 10 --warmup 3 --no-cpu-baseline --no-per-graph --e2e-streams 0 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
tail -1 $O/bench.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['per_step']
print('value',d['value'],'build',p['build_ms'],'solve',p['solve_ms'],'frac',d['roofline']['frac'],'parity',d.get('parity'))"
if [ -z "$NOLAUNCH" ]; then
  timeout 600 bash tools/build_profile.sh > /dev/null 2>&1; cp gpurun_out/bp/launches_${WL:-c5}_summary.txt $O/ 2>/dev/null
  head -30 $O/launches_${WL:-c5}_summary.txt
fi
