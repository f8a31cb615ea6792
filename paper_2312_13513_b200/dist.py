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

__all__ = ["shard", "GlobalReductions", "slab", "exchange_halos"]


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


def slab(nz_global: int, rank: int | None = None, world: int | None = None):
    """[z0, z1) planes of this rank's z-slab of a periodic box (NEXT-1 Laplacian consumer): contiguous,
    balanced, every rank at least one plane."""
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if world > nz_global:
        raise ValueError(f"{world} ranks for {nz_global} planes")
    return nz_global * rank // world, nz_global * (rank + 1) // world


def exchange_halos(bottom: torch.Tensor, top: torch.Tensor, group=None):
    """The halo exchange of the z-slab decomposition (NCCL peer-to-peer between GPUs, over
    NVLink/NVSwitch; gloo in the CPU tests): every rank sends its bottom plane to the rank below and its
    top plane to the rank above on the periodic ring, and receives (halo_lo, halo_hi) = (top plane of the
    rank below, bottom plane of the rank above).  Planes are the [(ns + 3)][nx ny] packs of
    rc_pack_planes.  One rank: the periodic wrap onto itself."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return top.clone(), bottom.clone()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    below, above = (rank - 1) % world, (rank + 1) % world
    lo, hi = torch.empty_like(top), torch.empty_like(bottom)
    # per peer, sends and receives are matched in posting order: my top is the halo_lo of the rank
    # above (posted first on both sides), my bottom the halo_hi of the rank below
    ops = [dist.P2POp(dist.isend, top, above, group), dist.P2POp(dist.isend, bottom, below, group),
           dist.P2POp(dist.irecv, lo, below, group), dist.P2POp(dist.irecv, hi, above, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return lo, hi
