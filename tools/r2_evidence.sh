#!/bin/bash
# Round-2 ncu / sanitizer evidence (one GPU).  Output under gpurun_out/r2e/.
#  1. same-capture traffic of k_solve (DRAM bytes, L2 hit, warp efficiency paired with each
#     launch's own counters) for C5, C3-hub20, C2 and C4 (SURVEY 8(d) "ncu evidence per kernel")
#  2. ncu --set full of one k_solve launch on C3-hub20, C2 and C4
#  3. compute-sanitizer memcheck / racecheck / synccheck / initcheck on small solves
O=gpurun_out/r2e
mkdir -p $O
for W in ${TRAFFIC:-c5 c3h c2 c4}; do
  timeout 900 python tools/traffic_run.py --workload $W --out $O/traffic_${W}_bcsr.json > $O/traffic_$W.log 2>&1
done
for W in ${FULL:-c3h c2 c4}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 3 -c 1 -o $O/full_${W}_k_solve \
      python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-per-graph --e2e-streams 0 > /dev/null 2>$O/full_${W}.err
  python tools/ncu_summary.py $O/full_${W}_k_solve.ncu-rep > $O/full_${W}_k_solve_summary.txt 2>&1
  rm -f $O/full_${W}_k_solve.ncu-rep   # (gpurun copies back <= 64 MiB)
done
for T in ${SAN:-memcheck racecheck synccheck initcheck}; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_run.py ${SANCASES:-} > $O/sanitizer_$T.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$T.txt
done
rm -f gpurun_out/traffic_*.csv gpurun_out/steps_*.json*
du -sh gpurun_out
