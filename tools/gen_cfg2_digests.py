"""Generate tests/golden/cfg2_level7_digests.json (TEST INFRASTRUCTURE).

Config 2's headline level 7 (214,990,848 tets) is refined by the CPU oracle
(oracle/phfem_oracle.c, bit-for-bit pinned to the reference's red_refine)
from the 6-Kuhn unit cube, and its connectivity is summarised by
or_conn_digests: SHA-256 of edge_nodes, edge_of_slot, faces, face_of_slot,
sigma, face_slots, face_area, face_class and multiplier_index computed in
one element-order pass with the reference's first-occurrence rules (the full
oracle tables need > 62 GB at this level, SURVEY.md 8(c) "Limits").  The
pass is checked against the full oracle tables at levels 0-5 by
tests/test_oracle_pins.py::test_streaming_digests_match_full_tables.
Also records the digests of levels 5 and 6 and of the refined level-7 mesh.

Usage: python tools/gen_cfg2_digests.py   (~40 GB of host memory, ~15 min)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bind import Oracle  # noqa: E402


def main(top=7):
    O = Oracle()
    m = O.kuhn(1, 1, 1, dmask=0x3F)
    out = {}
    for lv in range(top + 1):
        if lv >= 5:
            t0 = time.time()
            d = O.conn_digests(m)
            d.update(level=lv, ne=m.ne, nc=m.nc, nd=len(m.db), nn=len(m.nb), seconds=time.time() - t0,
                     mesh_coords=O.sha256(m.coords), mesh_tets=O.sha256(m.tets), mesh_db=O.sha256(m.db))
            out[f"level{lv}"] = d
            print(json.dumps(d), flush=True)
        if lv < top:
            m = O.refine(m)[0]
    with open(os.path.join(ROOT, "tests", "golden", "cfg2_level7_digests.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
