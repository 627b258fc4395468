"""Per-entry error of the load-vector data (rhs = B_T, rhs_neg, b_D) of the
GPU path against the CPU oracle, for each config (scaled and full size).

Prints one JSON line per case: the worst per-entry relative error
|g - o| / max(|o|, floor) with floor = 1e-12 ||o||_inf, and the count of
entries above 1e-12.  Used to set the per-entry bar of check_system.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bind import Oracle  # noqa: E402
from paper_2509_11133_b200 import configs  # noqa: E402
from paper_2509_11133_b200 import phfem as ph  # noqa: E402


def per_entry(g, o):
    fl = 1e-12 * (np.abs(o).max() if o.size else 0.0)
    r = np.abs(g - o) / np.maximum(np.abs(o), max(fl, 1e-300))
    i = int(np.argmax(r)) if r.size else 0
    return dict(worst=float(r.max()) if r.size else 0.0, n_gt_1e12=int((r > 1e-12).sum()),
                n_gt_1e13=int((r > 1e-13).sum()), q999=float(np.quantile(r, 0.999)) if r.size else 0.0,
                at=i, ref=float(o[i]) if r.size else 0.0, n=int(o.size))


def main(cases):
    O = Oracle()
    for cid, factor in cases:
        cfg = configs.CONFIGS[cid].scaled(factor) if factor > 1 else configs.CONFIGS[cid]
        m = O.kuhn(cfg.nx, cfg.ny, cfg.nz, lx=cfg.lx, ly=cfg.ly, lz=cfg.lz, jitter=cfg.jitter,
                   seed=configs.SEED_JITTER, dmask=cfg.dirichlet_mask)
        for _ in range(cfg.levels):
            m = O.refine(m)[0]
        k = cfg.coefficients(m.ne)
        g = ph.Mesh.from_arrays(m.coords, m.tets, m.db, m.nb, m.level)
        if k["a_elem"] is not None or k["a_diag"] is not None or cfg.c != 1.0:
            g.set_coefficients(k["a_elem"], k["a_diag"], cfg.c)
        fo = O.faces(m)
        so = O.assemble(m, fo, cfg.problem, cfg.c, k["a_elem"], k["a_diag"], with_c=False)
        sg = g.assemble(cfg.problem)
        out = {"config": cfg.name, "factor": factor, "ne": m.ne}
        rs, ns = O.entry_scales(m, fo, cfg.problem, cfg.c, k["a_elem"], k["a_diag"])
        for key in ("rhs", "rhs_neg", "bd"):
            out[key] = per_entry(sg[key], so[key])
        for key, sc in (("rhs", rs), ("rhs_neg", ns)):
            d = np.abs(sg[key] - so[key]) / np.maximum(np.maximum(sc, np.abs(so[key])), 1e-300)
            out[key]["componentwise_worst"] = float(d.max())
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    cs = [(1, 1), (3, 8), (4, 16), (5, 8), (3, 1), (5, 1)]
    if len(sys.argv) > 1:
        cs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]]
    main(cs)
