"""One connectivity pass of config 2's level 7 bracketed by
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2509_11133_b200 import phfem as ph  # noqa: E402

lv = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 7
m = ph.Mesh.kuhn(1, 1, 1, dirichlet_mask=0x3F)
for _ in range(lv):
    # classified before refining, as in bench.py --config 2: the child's
    # connectivity then follows from the parent's (refine_conn.cu)
    if "--generic" not in sys.argv:
        m.pipeline(0, do_refine=False, assemble=False)
    m.refine()
m.pipeline(0, do_refine=False, assemble=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st, _ = m.pipeline(0, do_refine=False, assemble=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: round(v, 3) for k, v in st.items()})
