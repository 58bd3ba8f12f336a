"""One warm EdaPass of a config (CFG env, default 4) after two untimed
passes -- the program a launch-list capture of a whole pass profiles."""
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
for _ in range(3):
    eng.run()
torch.cuda.synchronize()
print("ok")
