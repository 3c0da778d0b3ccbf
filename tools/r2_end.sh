#!/bin/bash
# End-of-session evidence (one GPU): default bench line, GPU tests, C5 launch list, workload trace.
O=gpurun_out/${TAG:-end}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 bash tools/build_profile.sh > /dev/null 2>&1; cp gpurun_out/bp/launches_c5_summary.txt $O/ 2>/dev/null
[ -n "$TRACE" ] && timeout 900 python tools/workload_trace.py > $O/workload_trace.md 2> $O/workload_trace.err
tail -3 $O/gpu_tests.txt; tail -1 $O/smoke.txt
