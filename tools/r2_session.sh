#!/bin/bash
# Session check on one GPU: default bench line (C5 + per-graph sub-lines + parity gate), then the GPU tests.
O=gpurun_out/${TAG:-s3}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.txt
tail -3 $O/gpu_tests.txt
