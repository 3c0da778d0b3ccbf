timeout 100 python tools/probe.py path20000 --reps 1 | python tools/summ.py
for mode in 0 1; do
for g in 0.5 1 2; do timeout 300 python tools/probe.py c4 c2r r18h r18p --reps 1 --beta 0.5 --gamma $g --mode $mode | python tools/summ.py "mode=$mode gamma=$g"; done
done
timeout 300 python tools/probe.py c3h c3p c2u --reps 1 --mode 1 | python tools/summ.py "mode=1 default"
timeout 300 python tools/probe.py c3h c3p c2r c4 --reps 1 --mode 1 --layout rcsr | python tools/summ.py "mode=1 rcsr"
