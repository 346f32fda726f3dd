"""Scenario sharding across GPUs (one process per GPU, torch.distributed).

Scenarios are independent units: rank r of N replays the contiguous global
ids [r*S/N, (r+1)*S/N) — the duration of every (task, scenario) is a pure
function of the global scenario id, so results do not depend on N.  The only
collective is the final gather of per-scenario results (span, per-rank
breakdown, per-stream busy) to rank 0; timestamps stay on each GPU.
"""
from __future__ import annotations


def shard(total: int, world: int, rank: int) -> tuple:
    """(first global scenario id, count) of this rank's shard."""
    if total % world:
        raise ValueError(f"{total} scenarios do not split evenly over {world} ranks")
    per = total // world
    return rank * per, per


def gather_rows(local, world: int, rank: int, out=None, root: int = 0):
    """Gather equally-sized per-scenario row blocks to `root` in rank order
    (global scenario order).  `out` (root only) has world * local.shape[0]
    rows.  Works with the nccl (device tensors) and gloo (CPU) backends."""
    import torch.distributed as dist
    if world == 1:
        if out is not None:
            out.copy_(local)
        return out
    parts = list(out.chunk(world)) if rank == root else None
    dist.gather(local, parts, dst=root)
    return out
