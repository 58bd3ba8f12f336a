"""One AD and one TL sweep over a BASELINE config's member block, after one
warm-up sweep each -- the program the per-config ncu capture profiles:

    python tools/sweep_ncu.py 4          # plain run first (must exit 0)
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
        --clock-control none -k regex:'k_ad|k_tl' -s <2 x chunks> -c <2 x chunks> --csv \
        --log-file gpurun_out/sweep_ncu_cfg4.csv python tools/sweep_ncu.py 4

tools/ncu_to_json.py folds the CSVs into profiles/r2_sweep_ncu.json, which
bench.py reads (roofline.traffic, fp64.executed_pipe_util_pct)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23571_b200 import build  # noqa: E402
build.build()
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = BASELINE_CONFIGS[cid]
dens = build_ensemble(cfg)
lin = dens.lin
M = cfg.members
ct = torch.arange(1, M + 1, dtype=torch.int32, device="cuda")
V = torch.randn(M, cfg.n, dtype=torch.float64, device="cuda")
W = torch.randn(M, lin.p, dtype=torch.float64, device="cuda")
for _ in range(2):  # warm-up, then the profiled sweeps
    lin.ad_cols(W, ct)
    lin.tl_cols(V, ct)
torch.cuda.synchronize()
chunks = -(-cfg.n_steps // 12) if cfg.n_steps > 12 else 1
print(f"sweep_ncu cfg{cid}: {M} columns, {chunks} launch(es) per sweep")
