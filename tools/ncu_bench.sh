#!/bin/bash
# launch list (per-kernel device time) of one bench step, and full captures of the top kernels
set -x
mkdir -p gpurun_out
WL=${WL:-c5}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL}.csv \
    python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_${WL}.json 2>gpurun_out/ncu_bench_${WL}.err
for K in ${KERNELS:-k_solve k_sort_warp k_mate k_scatter_bcsr}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/full_${WL}_$K \
      python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>gpurun_out/full_${WL}_$K.err
done
