mkdir -p gpurun_out/gs
for G in 0.25 0.5 1 2 4 8; do
  timeout 900 python tools/probe.py c2r c2u g256r c4 c3h --reps 3 --gamma $G 2>/dev/null | python tools/summ.py "g$G" >> gpurun_out/gs/gs.txt
done
