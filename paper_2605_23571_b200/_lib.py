"""ctypes binding of libedak.so (the C ABI in include/edak.h).

This module is the only place the host layer touches the native library.
There is no fallback: if the library is missing or fails to load, importing
it raises, and every GPU entry point in the package fails loudly.
"""

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libedak.so")

i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p


class Problem(C.Structure):
    """Mirror of ``edak_problem`` (include/edak.h)."""

    _fields_ = [
        ("n", i32), ("n_steps", i32), ("dt", f64), ("forcing", f64),
        ("states", vp), ("stages", vp), ("traj_stride", i64),
        ("stage_mode", i32), ("pad0", i32),
        ("gpos", vp), ("tpos", vp), ("G", i32), ("T", i32), ("sigma2", f64),
        ("taps", vp), ("ntaps", i32), ("tap_w", i32),
        ("os_spec", vp), ("os_tw", vp), ("os_logm", i32), ("pad1", i32),
    ]


_PROTOS = {
    "edak_version": (C.c_char_p, []),
    "edak_last_error": (C.c_char_p, []),
    "edak_launch_count": (i64, []),
    "edak_integrate": (C.c_int, [C.c_int, C.c_int, f64, f64, vp, C.c_int, vp, i64, vp, i64, vp]),
    "edak_tendency": (C.c_int, [C.c_int, C.c_int, vp, f64, vp, vp]),
    "edak_tendency_tlm": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp]),
    "edak_tendency_adj": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp]),
    "edak_axpy_rn": (C.c_int, [i64, vp, f64, vp, vp, vp]),
    "edak_rk4_combine": (C.c_int, [i64, vp, f64, vp, vp, vp, vp, vp, vp]),
    "edak_observe": (C.c_int, [vp, i64, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, vp, vp]),
    "edak_circ_apply": (C.c_int, [C.POINTER(Problem), vp, vp, C.c_int, vp]),
    "edak_sweep_work_doubles": (i64, [C.POINTER(Problem), C.c_int]),
    "edak_tl_sweep": (C.c_int, [C.POINTER(Problem), vp, vp, C.c_int, vp, vp, vp]),
    "edak_ad_sweep": (C.c_int, [C.POINTER(Problem), vp, vp, C.c_int, vp, vp, vp]),
    "edak_work_doubles": (i64, [C.POINTER(Problem), C.c_int]),
    "edak_hessian_block": (C.c_int, [C.POINTER(Problem), vp, vp, C.c_int, vp, f64, vp, vp, vp, vp]),
    "edak_hessian_dot_tiles": (i64, [C.c_int]),
    "edak_rhs": (C.c_int, [C.POINTER(Problem), vp, vp, C.c_int, vp, vp, vp]),
    "edak_cost": (C.c_int, [C.POINTER(Problem), vp, vp, vp, C.c_int, vp, vp, vp]),
    "edak_gemm_tn_partials": (i64, [C.c_int, C.c_int, i64]),
    "edak_gemm_tn": (C.c_int, [vp, i64, vp, i64, vp, C.c_int, C.c_int, C.c_int, i64, vp, vp]),
    "edak_gemm_nn": (C.c_int, [vp, i64, vp, C.c_int, vp, vp, i64, f64, vp, i64, i64, C.c_int,
                               C.c_int, vp]),
    "edak_potrf_shifted": (C.c_int, [vp, C.c_int, vp, C.c_int, f64, vp, vp, vp]),
    "edak_trinv_upper": (C.c_int, [vp, C.c_int, vp, vp]),
    "edak_svd_work_doubles": (i64, [C.c_int, C.c_int]),
    "edak_svd_jacobi": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
    "edak_pcg_work_doubles": (i64, [C.c_int, C.c_int]),
    "edak_pcg_init": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp]),
    "edak_pcg_cost0": (C.c_int, [C.c_int, C.c_int, vp, f64, vp, C.c_int, vp]),
    "edak_pcg_alpha": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp, C.c_int,
                                 vp]),
    "edak_pcg_lmp_beta": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, f64, vp, vp,
                                    C.c_int, vp, vp, C.c_int, vp]),
    "edak_pcg_beta": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp, f64, vp, vp, C.c_int, vp, vp,
                                C.c_int, vp]),
    "edak_lmp_work_doubles": (i64, [C.c_int, C.c_int, C.c_int]),
    "edak_chol_inv_work_doubles": (i64, [C.c_int]),
    "edak_pcg_small": (C.c_int, [C.POINTER(Problem), vp, C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, f64,
                                 vp, vp, vp, C.c_int, vp, vp, vp]),
    "edak_chol_inv": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, f64, vp, vp, vp, vp]),
    "edak_lmp_apply": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp]),
    "edak_col_dots": (C.c_int, [C.c_int, C.c_int, vp, vp, vp, vp]),
    "edak_peak_dfma": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "edak_peak_dmma": (C.c_int, [vp, C.c_int, C.c_int, vp]),
}

EXPORTED = tuple(_PROTOS)


def load(path=LIB_PATH):
    """dlopen libedak.so and attach prototypes; raises if anything is off."""
    if not os.path.exists(path):
        raise ImportError(
            f"libedak.so not found at {path}; build it with "
            "`python -m paper_2605_23571_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


class EdakError(RuntimeError):
    """A native entry point returned a non-zero status."""


def call(name, *args):
    """Call ``name`` and raise EdakError on a non-zero status."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().edak_last_error().decode(errors="replace")
        raise EdakError(f"{name} failed ({rc}): {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("edak entry points take CUDA tensors")
    return t.data_ptr()


def stream(s=None):
    """cudaStream_t of the current (or given) torch stream."""
    s = torch.cuda.current_stream() if s is None else s
    return s.cuda_stream


# kernels launched by CUDA-graph replays (the C counter sees a graph's
# launches once, at capture): krylov adds each replay's node count here
_GRAPH_LAUNCHES = [0]


def launch_count():
    """Our kernels launched so far: direct launches + graph-replayed ones."""
    return int(lib().edak_launch_count()) + _GRAPH_LAUNCHES[0]
