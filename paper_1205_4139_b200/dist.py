"""Multi-process plumbing for the sharded single-signal solver (config 5).

One process per GPU, each holding one `LargeShard`.  The shards exchange on
the device through NCCL inside fmp_large_group_solve (C ABI): per iteration
an all-gather of identification records and, before a conventional row, an
all-reduce of the residual's partial sums.  torch.distributed is used only
to hand the NCCL unique id from rank 0 to the others.
"""
from __future__ import annotations

import torch.distributed as dist

from . import Comm


def nccl_comm(device: int, group=None) -> Comm:
    """This rank's communicator over the torch.distributed group's ranks."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    return Comm.init_rank(device, world, rank, uid[0])


def gather_records(record: bytes, group=None) -> list:
    """All-gather of one record per rank (the host mirror of the device
    exchange; CPU tests run it over gloo)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, record, group=group)
    return out
