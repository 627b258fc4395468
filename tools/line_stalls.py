"""Warp-stall reasons per source line of one kernel in an .ncu-rep
(--import-source on; the object compiled with -lineinfo).

usage: python tools/line_stalls.py REP.ncu-rep OBJ.o MANGLED_SUBSTRING NCU_KERNEL_REGEX
"""
import sys, csv, subprocess, re, collections
sys.path.insert(0,'/root/repo/tools')
from line_hot import line_table
rep,obj,kern=sys.argv[1:4]
tabs=line_table(obj,kern); tab=tabs[sorted(tabs,key=len)[0]]
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","-k","regex:"+sys.argv[4],"-c","1"],capture_output=True,text=True).stdout
hdr=None;base=None
R=['stall_wait','stall_long_sb','stall_math','stall_selected','stall_not_selected','stall_dispatch','stall_short_sb','stall_branch_resolving','stall_no_inst','stall_drain','stall_lg']
agg=collections.defaultdict(lambda: collections.Counter())
for x in csv.reader(out.splitlines()):
    if x and x[0]=="Address": hdr=x; continue
    if not hdr or not x or x[0]=="Kernel Name": continue
    d=dict(zip(hdr,x))
    try: a=int(d["Address"],16)
    except: continue
    base=a if base is None else base
    loc=tab.get(a-base,("?",0))
    for r in R: agg[loc][r]+=float(d.get(r) or 0)
tot=collections.Counter()
for v in agg.values(): tot.update(v)
T=sum(tot.values())
print('TOTAL', {r: round(tot[r]/T*100,1) for r in R})
for loc,v in sorted(agg.items(), key=lambda kv:-sum(kv[1].values()))[:12]:
    s=sum(v.values()); print(f"{loc[0]}:{loc[1]} {s/T*100:.1f}%", {r.replace('stall_',''): round(v[r]/s*100) for r in R if v[r]/s>0.04})
