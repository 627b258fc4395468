"""Where the e2e step's time beyond the device step goes (config 4): per
step, host time in from_arrays_async / pipeline / release, and the device
time of the pass itself (events on the library stream), over N steps.
usage: python tools/e2e_gap.py [steps=20]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_11133_b200 import configs  # noqa: E402
from paper_2509_11133_b200 import phfem as ph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = configs.CONFIGS[4]
mesh = cfg.build()
coords, tets, db, nb = mesh.arrays()
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
hc, ht, hd, hn = pin(coords), pin(tets), pin(db), pin(nb)
stream = torch.cuda.ExternalStream(ph.stream_ptr())
for rep in range(2):
    nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn)
    tc, tp, tr, tw, sts = [], [], [], [], []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    w0 = time.perf_counter()
    for k in range(n):
        cur = nxt
        a = time.perf_counter()
        nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn) if k + 1 < n else None
        b0 = time.perf_counter()
        cur.sizes()  # waits for this mesh's upload (finish_upload)
        b = time.perf_counter()
        tw.append(b - b0)
        ev[k][0].record(stream)
        st, _ = cur.pipeline(cfg.problem, True)
        ev[k][1].record(stream)
        sts.append(st)
        c = time.perf_counter()
        del cur
        d = time.perf_counter()
        tc.append(b0 - a)
        tp.append(c - b)
        tr.append(d - c)
    e1.record(stream)
    e1.synchronize()
    wall = (time.perf_counter() - w0) / n * 1e3
    spans = [ev[k][0].elapsed_time(ev[k][1]) for k in range(n)]
    gaps = [ev[k][1].elapsed_time(ev[k + 1][0]) for k in range(n - 1)]
    med = {k: round(float(np.median([x[k] for x in sts[:-1]])), 3) for k in sts[0]}
    print(f"  stages with the next upload in flight (median): {med}")
    print(f"  device: pass span median {np.median(spans):.3f} ms, gap between passes median {np.median(gaps):.3f} ms")
    print(f"rep {rep}: e2e {e0.elapsed_time(e1) / n:.3f} ms/step (wall {wall:.3f}); host per step: create "
          f"{1e3 * np.mean(tc):.3f} ms, upload wait {1e3 * np.mean(tw[1:]):.3f} ms, pipeline {1e3 * np.mean(tp):.3f} ms (first {1e3 * tp[0]:.3f}, "
          f"median {1e3 * np.median(tp):.3f}), release {1e3 * np.mean(tr):.3f} ms; last pass stages "
          f"{ {k: round(v, 3) for k, v in st.items()} }", flush=True)
