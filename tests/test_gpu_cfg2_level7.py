"""Config 2's headline level: the 6-Kuhn unit cube refined 7 times (the first
level with >= 2e7 tets, 214,990,848 tets) on the B200, its refined mesh and
its whole connectivity (edge numbering, face numbering, sigma, face slots,
areas, classes, multiplier rows) compared with the CPU oracle through
SHA-256 digests (tests/golden/cfg2_level7_digests.json, made by
tools/gen_cfg2_digests.py with the one-pass restatement or_conn_digests,
itself checked against the full oracle tables in
test_oracle_pins.py::test_streaming_digests_match_full_tables).  Levels 5
and 6 are checked the same way.  Bit-exact is the bar (north_star)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ph = pytest.importorskip("paper_2509_11133_b200.phfem")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg2_level7_digests.json")


def _sha(a):
    h = hashlib.sha256()
    a = np.ascontiguousarray(a)
    mv = memoryview(a.reshape(-1).view(np.uint8))
    step = 1 << 28
    for i in range(0, len(mv), step):
        h.update(mv[i:i + step])
    return h.hexdigest()


def _check_level(g, want):
    c, t, d, _ = g.arrays()
    assert (g.sizes()[0], g.sizes()[1]) == (want["nc"], want["ne"])
    assert _sha(c) == want["mesh_coords"] and _sha(t) == want["mesh_tets"] and _sha(d) == want["mesh_db"]
    del c, t, d
    en, eos = g.edges()
    assert len(en) == want["ned"]
    assert _sha(en) == want["edge_nodes"], "edge_nodes"
    assert _sha(eos) == want["edge_of_slot"], "edge_of_slot"
    del en, eos
    f = g.faces()
    assert f["nf"] == want["nf"]
    assert f["n_dirichlet"] == want["nd"] and f["n_neumann"] == 0
    for k in ("faces", "face_of_slot", "sigma", "face_slots", "area", "face_class", "mrow"):
        assert _sha(f[k]) == want[k], k


def test_config2_levels_5_to_7_connectivity_digests():
    if not os.path.exists(GOLD):
        pytest.fail("missing tests/golden/cfg2_level7_digests.json (tools/gen_cfg2_digests.py)")
    with open(GOLD) as fh:
        gold = json.load(fh)
    g = ph.Mesh.kuhn(1, 1, 1, dirichlet_mask=0x3F)
    for lv in range(8):
        if f"level{lv}" in gold:
            _check_level(g, gold[f"level{lv}"])
        if lv < 7:
            g.refine()
    assert g.sizes()[1] == 214990848
