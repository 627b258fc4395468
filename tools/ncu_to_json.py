"""Extract per-kernel facts from ncu --set full captures into
profiles/ncu_kernels.json (read by bench.py for roofline.traffic).

usage: python tools/ncu_to_json.py OUT.json [--config=NAME] REP.ncu-rep[=profiles/summary.txt] ...
Each kernel keeps its first launch in the capture; names are shortened to
`name<T>` (namespace and argument list dropped).  --config tags the
following captures with the workload they ran (bench.py only uses a flop
count captured on its own config).
"""
import csv
import json
import re
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_inst",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1, "%": 0.01}


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
    name = re.sub(r"\((?:int|bool|long|unsigned int)\)", "", name)
    return name.split("(")[0]


def facts(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(out.stdout.splitlines()))
    head, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(head, r))
        k = short(d["Kernel Name"])
        if k in res:
            continue
        v = {}
        for m, key in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                u = units[head.index(m)]
                v[key] = float(d[m].replace(",", "")) * SCALE.get(u, 1)
        res[k] = {
            "dram_bytes": v.get("dram_read", 0) + v.get("dram_write", 0),
            "dram_read": v.get("dram_read"),
            "dram_write": v.get("dram_write"),
            "time_s": v.get("time"),
            "fp64_pipe_frac": v.get("fp64_pipe"),
            "warps_active_frac": v.get("warps_active"),
            "mem_throughput_frac": v.get("mem_throughput"),
            "registers": v.get("registers"),
            "warp_instructions": v.get("warp_inst"),
        }
    for k, flop in fp64_flops(rep).items():
        if k in res:
            res[k]["fp64_flop"] = flop
    return res


def fp64_flops(rep):
    """fp64 flops per kernel (first launch) from the SASS source page:
    predicated-on thread instructions, DFMA = 2, DMUL / DADD = 1."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True)
    res, cur, hdr = {}, None, None
    for x in csv.reader(out.stdout.splitlines()):
        if x and x[0] == "Kernel Name":
            k = short(x[1])
            cur = None if k in res else k
            if cur:
                res[cur] = 0.0
            continue
        if x and x[0] == "Address":
            hdr = x
            continue
        if cur and hdr:
            d = dict(zip(hdr, x))
            w = d.get("Source", "").split()
            if not w:
                continue
            op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
            n = float(d.get("Predicated-On Thread Instructions Executed") or 0)
            res[cur] += 2 * n if op == "DFMA" else (n if op in ("DMUL", "DADD") else 0)
    return {k: v for k, v in res.items() if v > 0}


def main():
    out = sys.argv[1]
    try:
        with open(out) as f:
            data = json.load(f)
    except (OSError, ValueError):
        data = {}
    config = None
    for arg in sys.argv[2:]:
        if arg.startswith("--config="):
            config = arg.split("=", 1)[1]
            continue
        rep, _, src = arg.partition("=")
        for k, v in facts(rep).items():
            v["source"] = src or rep
            if config:
                v["config"] = config
            data[k] = v
    with open(out, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
