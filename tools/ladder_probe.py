"""Stage times of the pipeline on the config-2 ladder levels 5-7."""
import sys

sys.path.insert(0, ".")
from paper_2509_11133_b200 import phfem as ph  # noqa: E402

m = ph.Mesh.kuhn(1, 1, 1, dirichlet_mask=0x3F)
for lv in range(8):
    if lv >= 5:
        for _ in range(2):
            st, counts = m.pipeline(ph.PROBLEM_SIN3, do_refine=False, assemble=lv < 7)
        print(lv, m.sizes()[1], {k: round(v, 3) for k, v in st.items()}, flush=True)
    if lv < 7:
        m.refine()
