"""Summarise an ncu --csv launch list: per-kernel time and DRAM bytes over
the last N launches (default: all)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
byid = collections.OrderedDict()
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    byid.setdefault(d["ID"], {"name": name})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ids = list(byid)
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(ids)
tot = collections.OrderedDict()
for i in ids[-n:]:
    v = byid[i]
    t = tot.setdefault(v["name"], [0.0, 0.0, 0.0, 0])
    t[0] += v.get("gpu__time_duration.sum", 0) / 1e6
    t[1] += v.get("dram__bytes_read.sum", 0) / 1e9
    t[2] += v.get("dram__bytes_write.sum", 0) / 1e9
    t[3] += 1
S = sum(v[0] for v in tot.values())
for k, (ms, r, w, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} x{c:<3d} {ms:8.3f} ms {100*ms/S:5.1f}%  R {r:6.3f} GB  W {w:6.3f} GB  {(r+w)/ms*1e3 if ms else 0:7.1f} GB/s")
print(f"{'total':28s}      {S:8.3f} ms over {min(n, len(ids))} launches")
