#!/bin/bash
# Round-2 final evidence (one GPU): launch list of the C5 step, ncu --set full of k_solve (C5),
# same-capture traffic for C5 / C3h / C2 / C4, sanitizers (both solve paths), default bench.
O=gpurun_out/r2f
mkdir -p $O
timeout 900 bash tools/build_profile.sh && cp gpurun_out/bp/launches_c5_summary.txt $O/ 
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 -o $O/full_c5_k_solve \
    python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-graph --e2e-streams 0 > /dev/null 2>$O/full_c5.err
python tools/ncu_summary.py $O/full_c5_k_solve.ncu-rep > $O/full_c5_k_solve_summary.txt 2>&1
rm -f $O/full_c5_k_solve.ncu-rep
for W in c5 c3h c2 c4; do
  timeout 900 python tools/traffic_run.py --workload $W --out $O/traffic_${W}_bcsr.json > $O/traffic_$W.log 2>&1
done
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 30 python tools/sanitize_run.py > $O/sanitizer_$T.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$T.txt
done
rm -f gpurun_out/traffic_*.csv gpurun_out/steps_*.json* gpurun_out/bp/full_build_source.csv.gz
du -sh gpurun_out
