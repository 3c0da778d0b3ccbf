
timeout 120 python tools/probe.py path20000 --reps 1 | python tools/summ.py
for mode in 0 1; do
for beta in 0.02 0.1 0.5; do timeout 300 python tools/probe.py c4 g256r c2r r18h --reps 1 --beta $beta --mode $mode | python tools/summ.py "mode=$mode beta=$beta"; done
done
timeout 300 python tools/probe.py c3h c3p --reps 1 --beta 0.5 --mode 1 | python tools/summ.py "mode=1"
