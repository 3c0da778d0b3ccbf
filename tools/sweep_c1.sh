for sm in 0 1; do for bfs in 0 1; do for b in 0 8; do
timeout 100 python tools/probe.py c1 --reps 3 --small $sm --bfs $bfs --blocks $b | tail -1 | python tools/summ.py "small=$sm bfs=$bfs blocks=$b" | awk '{print $1,$2,$3,$4,$5,$6,$7,$8,$9,$10,$11,$12,$13,$14,$15,$16,$17, $NF, $(NF-1), $(NF-2)}'
done; done; done
