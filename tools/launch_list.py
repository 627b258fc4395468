"""Print an ncu --csv launch list (time, DRAM bytes) in launch order."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, by = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        n = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        by.setdefault(d["ID"], {"name": n})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for i, v in by.items():
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    r = v.get("dram__bytes_read.sum", 0) / 1e6
    w = v.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:>4} {v['name'][:34]:34s} {t:9.1f} us  R {r:8.1f} MB  W {w:8.1f} MB  {(r + w) / t if t else 0:6.2f} TB/s")
