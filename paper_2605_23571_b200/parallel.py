"""Multi-GPU member sharding: one process per GPU.

Members (with their trajectories) are independent units, so a rank owns a
contiguous slice of member ids and runs its members' rhs, PCG and J traces
with no data-path collective.  The only exchange step is the sketch: Gamma's
columns b_j - b_0 come from the first ``ell`` member ids, wherever they live;
every rank writes the rows it owns into an (ell, n) buffer (zeros elsewhere)
and one all-reduce(SUM) over NCCL/NVLink -- exact, since x + 0 = x --
gives every rank the identical Gamma.  Each rank then builds the same
Nystrom LMP from the replicated control trajectory (deterministic kernels),
so no broadcast of S is needed.  Works on CPU tensors with gloo (tests).
"""

import torch
import torch.distributed as dist


def shard(total, world, rank, align=2):
    """(offset, count) of a contiguous slice of ``total`` units, in blocks of
    ``align`` units (the last rank takes the remainder).  align=2 keeps every
    member's column pairing in the overlap-save U_B (columns 2c, 2c + 1) the
    same on every rank count, so sharded passes are bit-identical."""
    blocks = -(-total // align)
    base, extra = divmod(blocks, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    offset = min(total, lo * align)
    return offset, min(total, hi * align) - offset


def gather_sketch_rows(local_rows, member_offset, ell, group=None):
    """Global rows [0, ell) of the member-ordered sketch.

    local_rows: (count, n) rows of member ids member_offset .. +count.
    Returns an (ell, n) tensor identical on every rank."""
    n = local_rows.shape[1]
    out = torch.zeros((ell, n), dtype=local_rows.dtype, device=local_rows.device)
    lo = max(0, member_offset)
    hi = min(ell, member_offset + local_rows.shape[0])
    if hi > lo:
        out[lo:hi] = local_rows[lo - member_offset: hi - member_offset]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def max_over_ranks(value, device, group=None):
    """Max of a float over ranks (timing: the slowest rank defines the step)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])


def sum_over_ranks(value, device, group=None):
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t[0])
