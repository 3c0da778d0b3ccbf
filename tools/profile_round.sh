#!/bin/bash
# Evidence for profiles/<round>: bench lines (C5 default + reference arm, C4, C3 paper rule and
# hub20), the ncu launch list of one C5 bench step, a full capture of k_solve (dram traffic,
# the bench roofline's `traffic`) and of the top construction kernels, per-config probes.
R=${R:-r1}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for W in c4 c3 c3h; do
  timeout 900 python bench.py --workload $W --steps 5 > $O/bench_$W.json 2> $O/bench_$W.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-streams 0 > /dev/null 2>&1
python tools/launches.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 3 -c 1 -o $O/full_c5_k_solve \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-streams 0 > /dev/null 2>&1
python tools/ncu_summary.py $O/full_c5_k_solve.ncu-rep > $O/full_c5_k_solve_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_merge_warp|k_inscatter|k_mate|k_edges|k_merge_thread" \
    -c 6 -o $O/full_c5_build python tools/probe.py c5 --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/full_c5_build.ncu-rep > $O/full_c5_build_summary.txt 2>&1
timeout 900 python tools/probe.py c1 c2u c2r c3p c3h c4 r18p r18h --reps 3 > $O/probe_bcsr.jsonl 2>&1
python tools/phase_summary.py $O/probe_bcsr.jsonl > $O/probe_bcsr_phases.txt 2>&1
timeout 1500 python tools/tc_vc_table.py --reps 3 > $O/tc_vc_table.md 2> $O/tc_vc_table.err
timeout 900 python tools/workload_trace.py > $O/workload_trace.md 2> $O/workload_trace.err
for G in 0.25 0.5 1 2; do
  timeout 600 python tools/probe.py c5 c4 c3h --reps 2 --gamma $G > $O/gamma_$G.jsonl 2>&1
done
