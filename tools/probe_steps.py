import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2605_23571_b200 import build
build.build()
from paper_2605_23571_b200.engine import EdaPass
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
cfg = BASELINE_CONFIGS[4]
dens = build_ensemble(cfg, members=cfg.members, member_offset=0)
eng = EdaPass(dens, member_offset=0, total_members=cfg.members, distributed=False)
os.environ["EDAK_PCG_GROUPS"] = sys.argv[1]
for _ in range(3):
    eng.run()
torch.cuda.synchronize()
for i in range(8):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record(); eng.run(); e.record(); torch.cuda.synchronize()
    print(i, f"{s.elapsed_time(e):.1f} ms gpu, {1e3*(time.perf_counter()-t0):.1f} wall, mem {torch.cuda.memory_reserved()/1e9:.2f} GB", flush=True)
