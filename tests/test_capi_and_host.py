"""CPU-side checks: the C-ABI library loads and exports every symbol
include/edak.h declares (no compute calls), the host layer refuses to run
without CUDA (no CPU fallback), and host-side helpers behave."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "edak.h")).read()
    return sorted(set(re.findall(r"\b(edak_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2605_23571_b200 import _lib, build
    build.build()
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) == set(declared)
    assert lib.edak_version().startswith(b"edak")


def test_problem_struct_layout_matches_header(tmp_path):
    """ctypes mirror of edak_problem == the C compiler's layout (gcc)."""
    import ctypes
    import subprocess
    from paper_2605_23571_b200._lib import Problem
    src = tmp_path / "lay.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "edak.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(edak_problem),'
                   ' offsetof(edak_problem,traj_stride), offsetof(edak_problem,sigma2),'
                   ' offsetof(edak_problem,taps), offsetof(edak_problem,tap_w));}')
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got == [ctypes.sizeof(Problem), Problem.traj_stride.offset, Problem.sigma2.offset,
                   Problem.taps.offset, Problem.tap_w.offset]


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2605_23571_b200.assim import MemberProblem
    from paper_2605_23571_b200.covariance import DiagonalNoise, gaussian_factor
    from paper_2605_23571_b200.model import Trajectory
    from paper_2605_23571_b200.obs import ObsNetwork
    traj = Trajectory(np.zeros((3, 40)), np.zeros((2, 4, 40)), 0.025, 8.0)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        MemberProblem(traj, ObsNetwork([0, 2], [1]), gaussian_factor(40, 0.8, 2.0),
                      DiagonalNoise(1.0), np.zeros(2))


def test_factor_taps_truncation():
    from paper_2605_23571_b200.covariance import GridCovFactor, factor_taps, gaussian_factor
    for n, L, w in [(1024, 8.0, 47), (16384, 16.0, 94), (262144, 32.0, 188)]:
        taps, tw = factor_taps(gaussian_factor(n, 0.8, L))
        assert tw == w and taps.size == 2 * w + 1
        assert np.allclose(taps, taps[::-1], rtol=0, atol=1e-15 * taps.max())  # symmetric to FFT noise
    taps, tw = factor_taps(GridCovFactor(40, 0.8, 6.0, 10))
    assert taps.size == 40  # full ring


def test_factor_dense_and_correlation():
    """covariance.py:49-56 -- the dense circulant equals the FFT apply, is
    symmetric, and the implied correlation has a unit diagonal."""
    from paper_2605_23571_b200.covariance import GridCovFactor
    ub = GridCovFactor(40, 0.8, 6.0, 10)
    d = ub.dense()
    v = np.random.default_rng(3).standard_normal(40)
    ref = np.fft.irfft(np.fft.rfft(v) * ub.symbol, n=40)
    assert np.allclose(d @ v, ref, rtol=0, atol=1e-13)
    assert np.allclose(d, d.T, rtol=0, atol=1e-15)
    assert abs(ub.correlation()[0] - 1.0) < 1e-12
    assert np.allclose((d @ d.T)[0] / 0.8 ** 2, ub.correlation(), rtol=0, atol=1e-13)


def test_position_maps_time_major():
    from paper_2605_23571_b200.obs import ObsNetwork, position_maps, strided_grid
    net = ObsNetwork(strided_grid(16384, 4096), list(range(3, 25, 3)))
    gpos, tpos = position_maps(net, 16384, 24)
    assert (gpos[::4] == np.arange(4096)).all() and (gpos[1::4] == -1).all()
    assert list(np.flatnonzero(tpos >= 0)) == list(range(3, 25, 3))
    net = ObsNetwork([7, 3, 0], [4, 0])  # unsorted grid and times keep their order
    gpos, tpos = position_maps(net, 10, 4)
    assert gpos[7] == 0 and gpos[3] == 1 and gpos[0] == 2 and tpos[4] == 0 and tpos[0] == 1
    with pytest.raises(ValueError):
        ObsNetwork([1, 1], [2])


def test_product_twin_streams_match_oracle():
    """The product's input builder draws exactly the reference streams."""
    from oracle.streams import substream as osub
    from paper_2605_23571_b200.twin import substream
    a = substream(0, "bg", 17).standard_normal(5)
    b = osub(0, "bg", 17).standard_normal(5)
    assert (a == b).all()


def test_overlap_save_tables_reproduce_the_tap_convolution():
    """covariance.os_tables (circ_os.cu's block spectrum in bit-reversed
    order, 1/M folded in): un-permuted and used in a numpy circular block
    convolution, the valid outputs equal the tap convolution
    out_i = sum_k taps[k] x[(i + w - k) mod n] (circ.cu), and the block
    sizes follow os_logm_for."""
    import numpy as np
    from paper_2605_23571_b200.covariance import os_logm_for, os_tables
    rng = np.random.default_rng(5)
    for n, K, w, logm in [(16384, 189, 94, 10), (9000, 61, 20, 10), (262144, 377, 188, 11)]:
        assert os_logm_for(n, K) == logm
        taps = rng.standard_normal(K)
        spec, tw = os_tables(taps, w, logm)
        M, V, L = 1 << logm, (1 << logm) - K + 1, K - 1 - w
        rev = np.array([int(format(j, f"0{logm}b")[::-1], 2) for j in range(M)])
        H = np.empty(M, complex)
        H[rev] = spec[0::2] + 1j * spec[1::2]
        assert np.allclose(tw[0::2] - 1j * tw[1::2], np.exp(2j * np.pi * np.arange(M) / (2 * M)), atol=1e-16)
        x = rng.standard_normal(n)
        i0 = n - V // 2  # a block that wraps the ring
        z = x[(i0 - L + np.arange(M)) % n]
        y = (np.fft.ifft(np.fft.fft(z) * H) * M)[L:L + V]
        i = (i0 + np.arange(V)) % n
        direct = sum(taps[k] * x[(i + w - k) % n] for k in range(K))
        assert np.abs(y.real - direct).max() <= 1e-13 * np.abs(direct).max()
    assert os_logm_for(40, 40) == 0 and os_logm_for(1024, 97) == 0 and os_logm_for(16384, 600) == 0
