"""A/B of the face-solve SpMV paths on the BASELINE configs: per config the
full Schur CG (bench's solve_timed) and a hash of Lambda from solve_faces.
Run once per mode: PHFEM_CG_SELL=1 (SELL copy) or unset (element-major).
usage: python tools/cg_ab.py [configs=3,5,4]"""
import hashlib
import os
import sys

sys.path.insert(0, ".")
from paper_2509_11133_b200 import configs  # noqa: E402

mode = "sell" if os.environ.get("PHFEM_CG_SELL", "0") != "0" else "em"
for cid in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,5,4").split(",")]:
    cfg = configs.CONFIGS[cid]
    m = cfg.build()
    m.pipeline(cfg.problem, False)
    r = m.solve_timed(cfg.problem, tol=cfg.tol)
    lam, st = m.solve_faces(cfg.problem, tol=cfg.tol)
    h = hashlib.sha256(lam.tobytes()).hexdigest()[:16]
    print(f"{mode} cfg{cid} it={r['iterations']} ms/it={r['ms_per_iteration']:.4f} cg_s={r['cg_ms']/1e3:.3f} "
          f"faces_it={st['iterations']} lambda_sha={h}", flush=True)
