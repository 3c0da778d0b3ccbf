#!/bin/bash
# direction-switch threshold sweep (experiment builds libwbpr_<v>.so): solve_ms per config
mkdir -p gpurun_out/sw
for V in default ${VARIANTS:-a7 a3 a1 b8 b64}; do
  if [ $V = default ]; then L=""; else L="WBPR_LIB=paper_2404_00270_b200/libwbpr_$V.so"; fi
  env $L timeout 600 python tools/probe.py c5 --gamma 0.5 --reps 5 > gpurun_out/sw/$V.c5.jsonl 2>/dev/null
  env $L timeout 600 python tools/probe.py c3p c3h c4 --reps 5 > gpurun_out/sw/$V.rest.jsonl 2>/dev/null
done
