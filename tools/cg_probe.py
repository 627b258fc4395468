"""A short config-4 face solve (for profiling the CG kernels); the
iteration cap ends it early, which the library reports as a stall."""
import sys

sys.path.insert(0, ".")
from paper_2509_11133_b200 import configs  # noqa: E402
from paper_2509_11133_b200 import phfem as ph  # noqa: E402

cfg = configs.CONFIGS[4]
m = cfg.build()
try:
    m.solve_faces(cfg.problem, tol=cfg.tol, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
except ph.SolverError as e:
    print("capped:", e)
