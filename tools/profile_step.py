"""One device-resident pipeline step (connectivity + assembly/condensation +
refinement) of a BASELINE config, bracketed by cudaProfilerStart/Stop for
ncu --profile-from-start off: the launch list and full captures of one step.

usage: python tools/profile_step.py [config=4]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2509_11133_b200 import configs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = configs.CONFIGS[cid]
m = cfg.build()
for _ in range(3):
    m.pipeline(cfg.problem, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st, _ = m.pipeline(cfg.problem, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print({k: round(v, 4) for k, v in st.items()})
