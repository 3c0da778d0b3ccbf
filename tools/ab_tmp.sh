mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/ab/t.txt 2>&1
for r in 1 2 3; do
  for V in default a7 a4; do
    if [ $V = default ]; then L=""; else L="WBPR_LIB=paper_2404_00270_b200/libwbpr_$V.so"; fi
    env $L timeout 300 python bench.py --no-per-graph --no-cpu-baseline --steps 20 > gpurun_out/ab/$V.$r.json 2>/dev/null
  done
done
for V in default a7 a4; do
  if [ $V = default ]; then L=""; else L="WBPR_LIB=paper_2404_00270_b200/libwbpr_$V.so"; fi
  env $L timeout 600 python tools/probe.py c3p c3h c4 c1 --reps 7 > gpurun_out/ab/$V.probe.jsonl 2>/dev/null
done
