"""Wall/device time of the parts of one EdaPass (rhs, sketch + Nystrom + LMP,
batched PCG) for a config (CFG env, default 4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.krylov import pcg_members  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
for _ in range(2):
    eng.run()
torch.cuda.synchronize()


def t(fn, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        r = fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, r


tr, B = t(lambda: eng.rhs())
tl, (G, approx, lmp) = t(lambda: eng.build_lmp(B))
tp, _ = t(lambda: pcg_members(eng.members, B[1:].contiguous(), eng.scfg, lmp, eng.cost))
tall, _ = t(lambda: eng.run())
print(f"{cfg.name}: rhs {tr:.2f} ms  sketch+nystrom+lmp {tl:.2f} ms  pcg {tp:.2f} ms "
      f"({tp / eng.iters:.3f} ms/it)  pass {tall:.2f} ms")
for i in range(4):
    ti, _ = t(lambda: eng.run(), reps=1)
    print(f"  run {i}: {ti:.2f} ms")
