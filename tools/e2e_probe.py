import time, sys, json
sys.path.insert(0, '.')
import torch
from paper_2509_11133_b200 import phfem as ph, configs
cfg = configs.CONFIGS[4]
m = cfg.build()
for _ in range(3): m.pipeline(cfg.problem, True)
coords, tets, db, nb = m.arrays()
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
hc, ht, hd, hn = pin(coords), pin(tets), pin(db), pin(nb)
for i in range(5):
    t0 = time.perf_counter()
    m2 = ph.Mesh.from_arrays(hc, ht, hd, hn)
    t1 = time.perf_counter()
    st, _ = m2.pipeline(cfg.problem, True)
    t2 = time.perf_counter()
    del m2
    t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.2f} ms  pipeline {1e3*(t2-t1):.2f} ms (device total {st['total']:.2f})  destroy {1e3*(t3-t2):.2f} ms", st)
# reuse one handle: pipeline only
for i in range(3):
    t1 = time.perf_counter(); st, _ = m.pipeline(cfg.problem, True); t2 = time.perf_counter()
    print(f"resident pipeline {1e3*(t2-t1):.2f} ms (device {st['total']:.2f})")
# double-buffered e2e loop as in bench.py, per-step wall and device totals
nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn)
for k in range(6):
    t0 = time.perf_counter()
    cur = nxt
    nxt = ph.Mesh.from_arrays_async(hc, ht, hd, hn)
    t1 = time.perf_counter()
    st, _ = cur.pipeline(cfg.problem, True)
    t2 = time.perf_counter()
    del cur
    t3 = time.perf_counter()
    print(f"e2e step: enqueue upload {1e3*(t1-t0):.2f} ms  pipeline {1e3*(t2-t1):.2f} ms (device {st['total']:.2f}: "
          + " ".join(f"{n} {st[n]:.2f}" for n in ('star', 'groups', 'number', 'classify', 'assemble', 'refine'))
          + f")  destroy {1e3*(t3-t2):.2f} ms")
