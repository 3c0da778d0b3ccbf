#!/bin/bash
# Diagnostics for the current round: phase-time breakdown per config, launch list of one
# bench step, full ncu captures of the build kernels.  Output under gpurun_out/diag/.
O=gpurun_out/diag
mkdir -p $O
timeout 900 python tools/probe.py c5 r18p r18h c3p c3h c4 --reps 3 > $O/probe.jsonl 2> $O/probe.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_mate|k_merge_warp|k_inscatter|k_sort_tile|k_edges}" -s ${SKIP:-0} -c ${CNT:-7} \
    -o $O/full_build python tools/probe.py c5 --reps 1 > /dev/null 2>$O/full_build.err
python tools/ncu_summary.py $O/full_build.ncu-rep > $O/full_build_summary.txt 2>&1
