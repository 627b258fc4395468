"""The closed-form rules of refine_conn.cu (first-occurrence edge slots and
face mates of a red-refined child from its parent's tables), stated in
Python by tools/refined_conn_proto.py, against the oracle's generic tables
of the refined mesh (CPU; the GPU kernel is checked against the oracle in
test_gpu_parity.py::test_refined_chain_with_faces and by the config-2
digests)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from oracle_bind import Oracle, cube5  # noqa: E402

proto = pytest.importorskip("refined_conn_proto")


@pytest.mark.parametrize("name", ["cube5", "kuhn1_mixed"])
def test_closed_form_rules_match_generic_tables(name):
    O = Oracle()
    m = cube5() if name == "cube5" else O.kuhn(1, 1, 1, jitter=0.1, dmask=0x5)
    for _ in range(2):
        eos, ef, sm = proto.generic_tables(O, m)
        a0 = proto.a0_table(m.tets, eos, int(eos.max()) + 1)
        child = O.refine(m)[0]
        _, ef_c, sm_c = proto.generic_tables(O, child)
        ef_p, sm_p = proto.refined_tables(m.tets, eos, ef, sm, a0)
        assert np.array_equal(ef_p, ef_c)
        assert np.array_equal(sm_p, sm_c)
        m = child
