#!/bin/bash
# Launch list of the build kernels (one C5 batch step) and a full capture of chosen build kernels.
# usage: KRE='k_merge2$' bash tools/build_profile.sh ; output under gpurun_out/bp/
O=gpurun_out/bp
mkdir -p $O
WL=${WL:-c5}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$WL.csv \
    python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline --no-per-graph --e2e-streams 0 > /dev/null 2>$O/launches.err
python tools/launches.py $O/launches_$WL.csv > $O/launches_${WL}_summary.txt 2>&1
rm -f $O/launches_$WL.csv
if [ -n "$KRE" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-1} -c ${CNT:-1} -o $O/full_build \
      python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline --no-per-graph --e2e-streams 0 > /dev/null 2>$O/full.err
  python tools/ncu_summary.py $O/full_build.ncu-rep > $O/full_build_summary.txt 2>&1
  ncu -i $O/full_build.ncu-rep --page source --csv > $O/full_build_source.csv 2>/dev/null
  gzip -f $O/full_build_source.csv
  rm -f $O/full_build.ncu-rep
fi
