import torch, time
for n, M in ((16384, 200), (16384, 100), (262144, 256)):
    Z = torch.randn(M, n, dtype=torch.float64, device="cuda")
    sym = torch.rand(n // 2 + 1, dtype=torch.float64, device="cuda")
    f = lambda: torch.fft.irfft(torch.fft.rfft(Z, dim=1) * sym, n=n, dim=1)
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    print(n, M, f"{s.elapsed_time(e)/10*1e3:.1f} us (rfft + mul + irfft, cuFFT via torch)")
