"""Data-parallel host plumbing: shard the batch, bootstrap the NCCL
communicator of libroast from a torch.distributed process group, all-reduce dM.

Under GMS every layer accumulates into the same dM, so data parallelism
is: split tokens / samples across ranks, replicate M, run the unchanged kernels on
each shard, sum dM over ranks once per step (roast_grad_allreduce), apply the same
update everywhere.  Only torch.distributed plumbing lives here; the exchange itself
is ncclAllReduce inside libroast.
"""
from __future__ import annotations


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous share of n items (sizes differ by at most 1)."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def broadcast_bytes(payload: bytes | None, rank: int, nbytes: int, group=None, device=None) -> bytes:
    """Rank 0's `payload` on every rank (e.g. the 128-byte NCCL unique id)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.tensor(list(payload), dtype=torch.uint8))
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().tolist())


def init_comm(ctx, rank: int, world: int, group=None, device=None) -> None:
    """Create libroast's NCCL communicator for this process group (no-op at world 1)."""
    from . import roast as R
    if world == 1:
        R.roast_comm_init(ctx.h, 0, 1, None)        # no communicator: the exchange is a no-op
        return
    uid = R.roast_comm_unique_id() if rank == 0 else bytes(128)
    uid = broadcast_bytes(uid, rank, 128, group=group, device=device)
    R.roast_comm_init(ctx.h, rank, world, uid)
