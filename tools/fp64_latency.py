"""DFMA throughput vs resident warps (latency hiding) on the box."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
lib = _lib.lib()
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
for blocks in (148, 296, 592, 1184):
    iters = 4096
    lib.edak_peak_dfma(sink.data_ptr(), 64, blocks, _lib.stream())
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.edak_peak_dfma(sink.data_ptr(), iters, blocks, _lib.stream())
    e.record()
    torch.cuda.synchronize()
    tf = 2.0 * 8 * iters * 256 * blocks / (s.elapsed_time(e) * 1e-3) / 1e12
    print(f"blocks {blocks:5d} ({blocks * 8 // 148} warps/SM, 8 indep chains/thread): {tf:6.2f} TFLOP/s",
          flush=True)
