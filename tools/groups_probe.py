"""A/B of pcg_members member groups (streams): step time with and without a
concurrent host thread, and the host-side launch time per pass."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
dens = build_ensemble(cfg)
eng = EdaPass(dens)


def bench(groups, reps=3):
    os.environ["EDAK_PCG_GROUPS"] = str(groups)
    eng.run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(reps):
        eng.run()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, (time.perf_counter() - t0) * 1e3 / reps


stop = False


def spin():
    while not stop:
        time.sleep(0.0005)


for g in (1, 2, 1, 2, 4):
    print(f"groups {g}: gpu {bench(g)[0]:.1f} ms  wall {bench(g)[1]:.1f} ms", flush=True)
th = threading.Thread(target=spin)
th.start()
for g in (1, 2):
    print(f"with thread, groups {g}: {bench(g)}", flush=True)
stop = True
th.join()

import subprocess  # noqa: E402
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.DEVNULL)
for g in (1, 2):
    print(f"with nvidia-smi -lms 100, groups {g}: {bench(g)}", flush=True)
p.terminate()
p.wait()
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False


def nvml_poll():
    while not stop:
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        time.sleep(0.1)


th = threading.Thread(target=nvml_poll)
th.start()
for g in (1, 2):
    print(f"with nvml 100 ms, groups {g}: {bench(g)}", flush=True)
stop = True
th.join()
