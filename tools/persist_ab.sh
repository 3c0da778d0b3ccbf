mkdir -p gpurun_out/pa
for R in 1 2; do
 for P in 0 1; do
  timeout 900 python tools/probe.py c5 --gamma 0.5 --reps 5 --persist $P 2>/dev/null | python tools/summ.py "p$P" >> gpurun_out/pa/pa.txt
  timeout 900 python tools/probe.py c3h c3p c4 --reps 5 --persist $P 2>/dev/null | python tools/summ.py "p$P" >> gpurun_out/pa/pa.txt
 done
done
