"""Device-array plumbing shared by the host layer.

Convention: a block of ``ncols`` ring vectors lives on the GPU as a
contiguous (ncols, n) float64 tensor -- column c contiguous -- which is the
transpose of the reference's numpy (n, ncols) blocks.  ``to_cols`` /
``from_cols`` convert at the drop-in boundary.
"""

import numpy as np
import torch

from . import _lib

F64 = torch.float64


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_23571_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _lib.lib()  # fail loudly if the native library is missing
    return torch.device("cuda", torch.cuda.current_device())


def to_cols(z, n):
    """numpy/torch (n,) or (n, l) -> (device (l, n) contiguous, was_vector,
    was_numpy)."""
    is_np = not isinstance(z, torch.Tensor)
    if is_np:
        a = np.asarray(z, dtype=float)
        vec = a.ndim == 1
        if a.shape[0] != n:
            raise ValueError(f"expected leading dimension {n}, got {a.shape}")
        cols = np.ascontiguousarray(a.reshape(n, -1).T)
        t = torch.from_numpy(cols).to(device(), non_blocking=False)
        return t, vec, True
    vec = z.dim() == 1
    if z.shape[0] != n:
        raise ValueError(f"expected leading dimension {n}, got {tuple(z.shape)}")
    t = z.to(device=device(), dtype=F64)
    t = t.reshape(n, -1).t().contiguous()
    return t, vec, False


def from_cols(t, vec, as_numpy):
    """(l, n) device block -> numpy/torch in the reference layout."""
    out = t[0] if vec else t.t()
    if as_numpy:
        return out.detach().cpu().numpy().copy() if not vec else out.detach().cpu().numpy()
    return out.contiguous()


def i32(a):
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=device())


def f64(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=device())
