"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel time of the LAST step.
usage: python tools/launches.py launches.csv [launches_per_step]"""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
def ms(d):
    v = float(d["Metric Value"]); u = d["Metric Unit"]
    return v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
# find step boundaries: a step starts at k_init_ctrl
starts = [i for i, d in enumerate(data) if "k_init_ctrl" in d["Kernel Name"]]
last = data[starts[-1]:] if starts else data
tot = collections.OrderedDict(); cnt = collections.Counter(); s = 0
for d in last:
    nm = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")[:50]
    v = ms(d); tot[nm] = tot.get(nm, 0) + v; cnt[nm] += 1; s += v
print(f"launches in last step: {len(last)}   total device time {s:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.3f} ms {100*v/s:5.1f}%  x{cnt[k]:<3d} {k}")
