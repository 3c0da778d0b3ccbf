#!/bin/bash
# Evidence for profiles/<round>: bench lines, ncu launch list, full capture of k_solve, per-config probes.
R=${R:-r1}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 3 -c 1 -o $O/full_c5_k_solve \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py $O/full_c5_k_solve.ncu-rep > $O/full_c5_k_solve_summary.txt 2>&1
for L in bcsr rcsr; do
  timeout 600 python tools/probe.py c1 c2u c2r c3p c3h c4 r18p r18h --reps 3 --layout $L > $O/probe_$L.jsonl 2>&1
  python tools/summ.py $L < $O/probe_$L.jsonl > $O/probe_${L}_summary.txt
done
