"""Per-kernel device time of one EdaPass (CFG env, default 4) from the CUDA
profiler API (torch.profiler/CUPTI; warm, the real multi-stream pass):
total and count per kernel name, sorted, plus the share of the pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
for _ in range(3):
    eng.run()
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "2"))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
phase = os.environ.get("PHASE", "pass")
B = eng.rhs()
fn = {"pass": eng.run, "nystrom": lambda: eng.build_lmp(B)}[phase]
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
wall = s.elapsed_time(e) * 1e3 / reps
rows = []
for ev in prof.key_averages():
    if ev.device_time_total > 0:
        rows.append((ev.device_time_total / reps, ev.count // reps, ev.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"{cfg.name}: {phase} {wall / 1e3:.2f} ms (events); summed kernel time {tot / 1e3:.2f} ms")
for us, cnt, name in rows[:25]:
    print(f"  {us / 1e3:8.3f} ms {100 * us / wall:5.1f}%  x{cnt:5d}  {name[:90]}")
