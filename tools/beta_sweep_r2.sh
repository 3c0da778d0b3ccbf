mkdir -p gpurun_out/bs
for B in 0.25 0.5 1 2 4; do
  timeout 900 python tools/probe.py c4 c3h c2u --reps 3 --beta $B 2>/dev/null | python tools/summ.py "b$B" >> gpurun_out/bs/bs.txt
  timeout 900 python tools/probe.py c5 --gamma 0.5 --reps 3 --beta $B 2>/dev/null | python tools/summ.py "b$B" >> gpurun_out/bs/bs.txt
done
