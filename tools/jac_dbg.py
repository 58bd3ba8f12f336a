import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_23571_b200.linalg import svd_jacobi, last_svd_sweeps
rng = np.random.default_rng(0)
rows, cols, v = (int(a) for a in sys.argv[1:4])
m = rng.standard_normal((rows, cols))
U, s, V = svd_jacobi(torch.tensor(m.T.copy(), device="cuda"), want_v=bool(v))
torch.cuda.synchronize()
print(rows, cols, v, os.environ.get("EDAK_JACOBI_SINGLE"), os.environ.get("EDAK_JACOBI_CLUSTER"), "ok",
      np.abs(s.cpu().numpy() - np.linalg.svd(m, compute_uv=False)).max(), last_svd_sweeps(), flush=True)
