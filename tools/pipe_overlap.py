"""Do the fp64 FMA pipe (DFMA) and the fp64 tensor pipe (DMMA) run
concurrently?  Time the two peak loops alone and on two streams at once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
lib = _lib.lib()
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
blocks = 148 * 4
it_f, it_m = 8192, 2048


def run(which):
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    if "f" in which:
        with torch.cuda.stream(s1):
            lib.edak_peak_dfma(sink.data_ptr(), it_f, blocks, _lib.stream())
    if "m" in which:
        with torch.cuda.stream(s2):
            lib.edak_peak_dmma(sink.data_ptr(), it_m, blocks, _lib.stream())
    torch.cuda.synchronize()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en)


for w in ("f", "m", "fm", "f", "m", "fm"):
    print(w, f"{run(w):.3f} ms", flush=True)
