"""Full BASELINE.json sizes against the CPU oracle, element for element.

Configs 3 and 5 (1.57M tets each: jittered Kuhn 64^3 x 6 with log-uniform
per-element diffusion; anisotropic 256 x 32 x 32 box with per-element
tensor choice) at their full size, and the config-4 mesh (12.6M tets) for
connectivity and the condensed system:

* the mesh from the device generator equals the oracle's bit for bit;
* edge and face tables (edge_nodes, edge_of_slot, faces, face_of_slot,
  sigma, face_slots, classes, multiplier rows, areas) bit-exact;
* element blocks A_T, C_T coefficients and rows, the SELL-32 Schur matrix S
  bit-exact; load vectors B_T, rhs_neg and b_D within 1e-12 relative (max
  norm) for the transcendental data (libdevice vs libm, economised series);
* one red refinement of the full mesh bit-exact (configs 3 and 5);
* config 2's ladder: the refined meshes of levels 6 and 7 (215M tets) and
  the connectivity of level 6 bit for bit.

The face solve itself is compared at scaled sizes in test_gpu_parity.py
(the oracle's serial CG would take tens of minutes here).  The module
takes ~2.5 min on the GPU box (oracle on one host core; ~20 GB of host
memory at config 4).
"""
import numpy as np
import pytest

from test_gpu_parity import check_connectivity, check_system, from_gpu

pytestmark = pytest.mark.gpu

ph = pytest.importorskip("paper_2509_11133_b200.phfem")
from paper_2509_11133_b200 import configs  # noqa: E402


def _pair(oracle, cid):
    cfg = configs.CONFIGS[cid]
    m = oracle.kuhn(cfg.nx, cfg.ny, cfg.nz, lx=cfg.lx, ly=cfg.ly, lz=cfg.lz, jitter=cfg.jitter,
                    seed=configs.SEED_JITTER, dmask=cfg.dirichlet_mask)
    g = cfg.build()
    mg = from_gpu(g)
    for k in ("coords", "tets", "db", "nb"):
        assert np.array_equal(getattr(mg, k), getattr(m, k)), k
    return cfg, m, g


@pytest.mark.parametrize("cid", [3, 5])
def test_full_size_connectivity_system_refinement(oracle, cid):
    cfg, m, g = _pair(oracle, cid)
    assert cfg.levels == 0 and m.ne == 1572864
    k = cfg.coefficients(m.ne)
    fo = check_connectivity(g, m, oracle)
    check_system(g, m, fo, oracle, cfg.problem, cfg.c, k["a_elem"], k["a_diag"])
    # one red refinement of the full mesh
    mo = oracle.refine(m)[0]
    g.refine()
    mg = from_gpu(g)
    for key in ("coords", "tets", "db", "nb"):
        assert np.array_equal(getattr(mg, key), getattr(mo, key)), key


def test_full_size_config4_connectivity_system(oracle):
    cfg, m, g = _pair(oracle, 4)
    assert m.ne == 12582912
    k = cfg.coefficients(m.ne)
    fo = check_connectivity(g, m, oracle)
    check_system(g, m, fo, oracle, cfg.problem, cfg.c, k["a_elem"], k["a_diag"])


def test_config2_levels_6_and_7(oracle):
    """Config 2's ladder (one cube -> 6 Kuhn tets, red refinement) past the
    level-5 check of test_gpu_parity.py: the refined meshes of levels 6
    (17.9M tets) and 7 (215M tets, the first level with >= 2e7 tets) bit for
    bit, and the full edge and face tables of level 6 (the
    oracle holds level 7's mesh but not its connectivity in a test)."""
    m = oracle.kuhn(1, 1, 1, dmask=0x3F)
    g = ph.Mesh.kuhn(1, 1, 1, dirichlet_mask=0x3F)
    for _ in range(6):
        m = oracle.refine(m)[0]
        g.refine()
    assert m.ne == 17915904
    mg = from_gpu(g)
    for k in ("coords", "tets", "db", "nb"):
        assert np.array_equal(getattr(mg, k), getattr(m, k)), k
    del mg
    check_connectivity(g, m, oracle)
    m7 = oracle.refine(m)[0]
    del m
    g.refine()
    assert m7.ne == 214990848
    mg = from_gpu(g)
    for k in ("coords", "tets", "db", "nb"):
        assert np.array_equal(getattr(mg, k), getattr(m7, k)), k
