"""Launch list driver for one Nystrom + LMP build of a config (CFG env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
B = eng.rhs()
eng.build_lmp(B)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.build_lmp(B)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
