"""A/B of whole EdaPass passes under environment variants (CFG env, default 4).

    python tools/ab_pass.py "" "EDAK_PCG_GROUPS=1" "EDAK_LMP_NN=0+EDAK_LMP_TN=0"

Each argument is a "+"-separated set of assignments applied before the pass
(the library and host layer read these knobs at launch time).  Prints the
median / min pass time over REPS passes (two interleaved rounds) and whether
the member increments are bit-identical to the first variant's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
reps = int(os.environ.get("REPS", "5"))
variants = sys.argv[1:] or [""]
keys = {kv.split("=")[0] for v in variants for kv in v.split("+") if kv}
times = {v: [] for v in variants}
ref = None
same = {}
for rnd in range(2):
    for v in variants:
        for k in keys:
            os.environ.pop(k, None)
        for kv in v.split("+"):
            if kv:
                a, b = kv.split("=", 1)
                os.environ[a] = b
        eng.members.__dict__.pop("_pcg_graphs", None)  # re-capture under this variant
        r = eng.run()
        torch.cuda.synchronize()
        x = r.x.cpu().numpy()
        if ref is None:
            ref = x
        same[v] = bool(np.array_equal(x, ref))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(reps):
            s.record()
            eng.run()
            e.record()
            torch.cuda.synchronize()
            times[v].append(s.elapsed_time(e))
for v in variants:
    t = np.array(times[v])
    print(f"{cfg.name} [{v or 'default'}]: median {np.median(t):.2f} ms  min {t.min():.2f} ms  "
          f"bit-identical x: {same[v]}")
