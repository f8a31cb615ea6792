"""Multi-GPU plumbing for the cell-local update.

Cells are independent: each rank owns the 128-aligned block rc_partition gives
it and runs rc_step on it with no data-path collective.  The only exchange per
time step is step a6, the global reductions: T_max (MAX) and the heat-release
sum plus the diagnostic counters (SUM), through torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests).
"""
import torch
import torch.distributed as dist

from ._rc import rc_partition

__all__ = ["shard", "GlobalReductions"]


def shard(n_global: int, rank: int | None = None, world: int | None = None):
    """[begin, end) of this rank's cells (rc_partition: contiguous, 128-aligned, balanced)."""
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return rc_partition(int(n_global), int(rank), int(world))


class GlobalReductions:
    """a6 across ranks, in place on the rc_cells reduction buffers.

    red  float64[2] = [max T, sum qdot V] of this rank (rc_step output)
    diag int64[5]   = per-rank counters (DIAG_NAMES)
    After the call every rank holds the global values.  Two collectives per
    step: one MAX of 8 bytes and one SUM of 48 bytes (counters travel as
    float64, exact below 2^53).
    """

    def __init__(self, device, group=None):
        self.group = group
        self.buf = torch.zeros(6, dtype=torch.float64, device=device)

    def __call__(self, red: torch.Tensor, diag: torch.Tensor):
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return red, diag
        dist.all_reduce(red[:1], op=dist.ReduceOp.MAX, group=self.group)
        self.buf[0:1].copy_(red[1:2])
        self.buf[1:].copy_(diag.to(torch.float64))
        dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
        red[1:2].copy_(self.buf[0:1])
        diag.copy_(self.buf[1:].to(torch.int64))
        return red, diag
