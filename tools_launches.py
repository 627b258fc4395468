"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
tail = data[-n:]
tot = collections.OrderedDict()
for d in tail:
    k = d['Kernel Name'].split('(')[0].replace('<unnamed>::', '').replace('void ', '')
    tot[k] = tot.get(k, 0) + float(d['Metric Value']) / 1e6
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {v:8.3f} ms  {100*v/s:5.1f}%")
print(f"{'total':40s} {s:8.3f} ms over {len(tail)} launches")
