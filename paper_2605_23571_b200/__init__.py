"""B200-native (sm_100a) engine for the Gauss-Newton 4D-Var Hessian block and
the spectral-LMP preconditioned CG of arxiv/paper_2605_23571 ("edasketch").

Drop-in modules mirror the reference package layout (pkg/src/edasketch):
``model``, ``covariance``, ``obs``, ``assim``, ``sketch``, ``nystrom``,
``lmp``, ``krylov``.  The compute path is libedak.so (csrc/, C ABI in
include/edak.h) called through ctypes; importing the GPU entry points
without the built library or without a CUDA device raises.
"""

__version__ = "0.1.0"
