"""Per-source-line profile of one kernel: joins the SASS page of an .ncu-rep
(--import-source on) with nvdisasm's line table of the cubin it ran.

usage: python tools/line_hot.py REP.ncu-rep OBJ.o KERNEL_SUBSTRING [N [DEPTH]]
DEPTH d attributes inlined code to the call frame d levels below the
kernel body (default: the innermost source line).
Prints, for the N hottest source lines (by warp-stall samples): samples,
fp64 flops (DFMA = 2), executed warp instructions.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel, depth=None):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
        cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        out = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cubin)], capture_output=True,
                             text=True, check=True).stdout
    table, cur, loc, chain = {}, None, None, []
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur = m.group(1) if kernel in m.group(1) else None
            continue
        if cur is None:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            chain.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            if chain:
                # chain: innermost frame first, the kernel body last
                loc = chain[0] if depth is None else chain[max(0, len(chain) - 1 - depth)]
                chain = []
            if loc:
                table.setdefault(cur, {})[int(m.group(1), 16)] = loc
    return table


def main():
    rep, obj, kernel = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    depth = int(sys.argv[5]) if len(sys.argv) > 5 else None
    tabs = line_table(obj, kernel, depth)
    fn = sorted(tabs, key=len)[0]
    tab = tabs[fn]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + re.match(r"[a-z_0-9]+", kernel).group(0),
                          "-c", "1"], capture_output=True, text=True).stdout
    hdr, base, agg = None, None, collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for x in csv.reader(out.splitlines()):
        if x and x[0] == "Address":
            hdr = x
            continue
        if not hdr or not x or x[0] == "Kernel Name":
            continue
        d = dict(zip(hdr, x))
        try:
            addr = int(d["Address"], 16)
        except ValueError:
            continue
        base = addr if base is None else base
        addr -= base  # ncu prints load addresses; the first row is the entry
        loc = tab.get(addr, ("?", 0))
        w = d.get("Source", "").split()
        op = (w[1] if w and w[0].startswith("@") else (w[0] if w else "")).split(".")[0]
        ti = float(d.get("Predicated-On Thread Instructions Executed") or 0)
        a = agg[loc]
        a[0] += float(d.get("Warp Stall Sampling (All Samples)") or 0)
        a[1] += 2 * ti if op == "DFMA" else (ti if op in ("DMUL", "DADD") else 0)
        a[2] += float(d.get("Instructions Executed") or 0)
    tot = [sum(v[i] for v in agg.values()) for i in range(3)]
    print(f"{fn}\n total samples {tot[0]:.0f}  fp64 flop {tot[1]:.3e}  warp inst {tot[2]:.3e}")
    for loc, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{loc[0]}:{loc[1]:<5d} samples {v[0] / tot[0] * 100:5.1f}%  fp64 {v[1] / max(tot[1], 1) * 100:5.1f}%  "
              f"inst {v[2] / tot[2] * 100:5.1f}%")


if __name__ == "__main__":
    main()
