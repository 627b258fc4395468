"""A short face solve of config 4 (or argv[2]) for profiling the CG
kernels; the iteration cap ends it early, which the library reports as a
stall.  usage: python tools/cg_probe.py [iterations=64] [config=4]"""
import sys

sys.path.insert(0, ".")
from paper_2509_11133_b200 import configs  # noqa: E402
from paper_2509_11133_b200 import phfem as ph  # noqa: E402

cfg = configs.CONFIGS[int(sys.argv[2]) if len(sys.argv) > 2 else 4]
m = cfg.build()
try:
    m.solve_faces(cfg.problem, tol=cfg.tol, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
except ph.SolverError as e:
    print("capped:", e)
