"""Time whole EdaPass passes (CFG env, default 4) with a given libedak build:

    python tools/time_pass.py [path/to/libedak.so]

Used to A/B compile-time variants (tools/build_exp.sh builds): prints the
median / min pass time over REPS passes and a checksum of the increments."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
    _lib._LIB = _lib.load(_lib.LIB_PATH)
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
reps = int(os.environ.get("REPS", "6"))
for _ in range(3):
    r = eng.run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = eng.run()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
x = r.x.cpu().numpy()
print(f"{cfg.name} [{sys.argv[1] if len(sys.argv) > 1 else 'in-tree'}]: median {np.median(ts):.2f} ms  "
      f"min {min(ts):.2f} ms  |x| {np.linalg.norm(x):.15e}  J_last[0] {r.traces[0].cost[-1]:.15e}")
