"""cfg1/cfg2: the persistent small-ring solve -- kernel-only device time vs
the whole pcg_members call (trace assembly on the host included)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2605_23571_b200 import _lib, krylov  # noqa: E402
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

for c in (1, 2):
    cfg = BASELINE_CONFIGS[c]
    eng = EdaPass(build_ensemble(cfg))
    eng.run()
    B = eng.rhs()
    _, _, lmp = eng.build_lmp(B)
    Bm = B[1:].contiguous()
    ens = eng.members
    sp = lmp.single_pass()
    orig = _lib.call
    reps = 20
    ev = []

    def timed(name, *a):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = orig(name, *a)
        e.record()
        ev.append((name, s, e))
        return r
    krylov._lib.call = timed
    for _ in range(3):
        krylov.pcg_members(ens, Bm, eng.scfg, lmp, eng.cost)
    torch.cuda.synchronize()
    ev.clear()
    t0 = time.perf_counter()
    for _ in range(reps):
        krylov.pcg_members(ens, Bm, eng.scfg, lmp, eng.cost)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    krylov._lib.call = orig
    k = [s.elapsed_time(e) for (n, s, e) in ev if n == "edak_pcg_small"]
    print(f"cfg{c}: members {ens.M} iters {eng.scfg.max_iters}: kernel {sum(k) / len(k):.3f} ms "
          f"({sum(k) / len(k) / eng.scfg.max_iters * 1e3:.1f} us/it), pcg_members wall {wall:.3f} ms", flush=True)
    # build_lmp breakdown
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(reps):
        eng.build_lmp(B)
    e.record()
    torch.cuda.synchronize()
    print(f"   build_lmp device {s.elapsed_time(e) / reps:.3f} ms wall {(time.perf_counter() - t0) / reps * 1e3:.3f} ms")
