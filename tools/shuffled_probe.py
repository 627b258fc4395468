"""Config 4's step on the same mesh with its nodes renumbered and its
elements shuffled (seeded): how much the kernels rely on the generator's
element / node locality.  usage: python tools/shuffled_probe.py [steps=10]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_11133_b200 import configs  # noqa: E402
from paper_2509_11133_b200 import phfem as ph  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = configs.CONFIGS[4]
stream = torch.cuda.ExternalStream(ph.stream_ptr())


def timed(m):
    for _ in range(3):
        m.pipeline(cfg.problem, True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        st, _ = m.pipeline(cfg.problem, True)
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / steps, st


m0 = cfg.build()
ms0, st0 = timed(m0)
c, t, d, n = m0.arrays()
rng = np.random.default_rng(7)
pn = rng.permutation(len(c)).astype(np.int32)
inv = np.argsort(pn)
pe = rng.permutation(len(t))
for name, (cc, tt, dd, nn) in {
    "elements shuffled": (c, t[pe], d, n),
    "nodes renumbered + elements shuffled": (c[inv], pn[t][pe], pn[d], pn[n]),
}.items():
    m = ph.Mesh.from_arrays(np.ascontiguousarray(cc), np.ascontiguousarray(tt, dtype=np.int32),
                            np.ascontiguousarray(dd, dtype=np.int32), np.ascontiguousarray(nn, dtype=np.int32))
    ms, st = timed(m)
    print(f"{name}: {ms:.3f} ms/step (generator order {ms0:.3f}); stages "
          f"{ {k: round(v, 3) for k, v in st.items()} }", flush=True)
print(f"generator order stages { {k: round(v, 3) for k, v in st0.items()} }")
