"""Opcode histogram and hottest SASS lines of the first kernel (or the
kernel whose name contains argv[2]) in an .ncu-rep captured with
--import-source on."""
import collections
import csv
import subprocess
import sys


def load(path, name=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    blocks, cur, hdr, kname = [], None, None, None
    for x in csv.reader(out.splitlines()):
        if x and x[0] == "Kernel Name":
            kname = x[1]
            cur = []
            blocks.append((kname, cur))
            continue
        if x and x[0] == "Address":
            hdr = x
            continue
        if cur is not None and hdr:
            cur.append(dict(zip(hdr, x)))
    for k, rows in blocks:
        if name is None or name in k:
            return k, rows
    raise SystemExit("kernel not found")


def main():
    k, rows = load(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
    print(k[:120])
    op, st = collections.Counter(), collections.Counter()
    te = ts = 0
    for r in rows:
        words = r["Source"].split()
        o = words[1] if words[0].startswith("@") else words[0]
        o = o.split(".")[0]
        e = int(r["Instructions Executed"] or 0)
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        op[o] += e
        st[o] += s
        te += e
        ts += s
    print(f"instructions {te}  stall samples {ts}")
    for o, c in op.most_common(16):
        print(f"  {o:10s} inst {c:12d} {c / te:6.1%}  samples {st[o] / max(ts, 1):6.1%}")
    print("hottest lines by samples:")
    for i, r in sorted(enumerate(rows), key=lambda p: -int(p[1]["Warp Stall Sampling (All Samples)"] or 0))[:15]:
        print(f"  {i:5d} {r['Source'].strip()[:60]:60s} exec {r['Instructions Executed']:>10s} samples {r['Warp Stall Sampling (All Samples)']}")


if __name__ == "__main__":
    main()


def stall_lines(path, name=None, n=25):
    """Hottest lines with their dominant stall reasons."""
    k, rows = load(path, name)
    reasons = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    for i, r in sorted(enumerate(rows), key=lambda p: -int(p[1]["Warp Stall Sampling (All Samples)"] or 0))[:n]:
        top = sorted(((int(r[c] or 0), c[6:]) for c in reasons), reverse=True)[:3]
        print(f"  {i:5d} {r['Source'].strip()[:50]:50s} {r['Warp Stall Sampling (All Samples)']:>6s} "
              + " ".join(f"{c}={v}" for v, c in top if v))
