#!/bin/bash
# A/B of experiment builds on one box: default libwbpr.so vs libwbpr_<V>.so, interleaved reps.
# usage: VARIANTS="eager" REPS=3 CFGS="c3h c4 c2u" bash tools/ab.sh ; output gpurun_out/ab/
O=gpurun_out/ab; mkdir -p $O
for R in $(seq 1 ${REPS:-3}); do
  for V in default ${VARIANTS}; do
    if [ $V = default ]; then L=""; else L="WBPR_LIB=paper_2404_00270_b200/libwbpr_$V.so"; fi
    env $L timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-per-graph --e2e-streams 0 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['per_step']; print('$V', 'rep$R', 'c5', 'value', d['value'], 'build', p['build_ms']['median'], 'solve', p['solve_ms']['median'], 'frac', d['roofline']['frac'])" >> $O/ab.txt
    if [ -n "${CFGS}" ]; then
      env $L timeout 600 python tools/probe.py ${CFGS} --reps 5 2>/dev/null | python tools/summ.py "$V rep$R" >> $O/ab.txt
    fi
  done
done
cat $O/ab.txt
