"""Multi-GPU plumbing for the lane-sharded IDM hot path.

Lanes are independent units (a vehicle reacts only to its leader in the same
lane; no lane changes), so ranks own contiguous whole-lane ranges and never exchange state.
Per optimizer step the only collective sums the Eq. 4 loss (L = sum_i L_i)
and, in shared-parameter mode, the six parameter gradients: ONE all-reduce of 7 fp64 values
(NCCL over NVLink on the GPU path; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_lanes(n_lanes: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous whole-lane range [l0, l1) of `rank`; boundaries are multiples of `align`
    lanes (except the last), shards differ by at most `align` lanes."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    chunks = (n_lanes + align - 1) // align
    c0 = chunks * rank // world
    c1 = chunks * (rank + 1) // world
    return min(n_lanes, c0 * align), min(n_lanes, c1 * align)


def reduce_step(loss: torch.Tensor, shared_grads: torch.Tensor | None = None, group=None):
    """Sum the loss (fp64 [1]) and optionally the shared gradients ([6], any float dtype)
    over all ranks, in place, with one all-reduce.  No-op when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    if shared_grads is None:
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)
        return
    buf = torch.empty(7, dtype=torch.float64, device=loss.device)
    buf[:1].copy_(loss)
    buf[1:].copy_(shared_grads.reshape(-1))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    loss.copy_(buf[:1])
    shared_grads.reshape(-1).copy_(buf[1:])


def max_over_ranks(x: float, device, group=None) -> float:
    """Max of a per-rank scalar (device timing: the slowest rank defines the step)."""
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(group=None):
    """dist.barrier() when distributed, else nothing."""
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)
