"""Multi-GPU plumbing for the lane-sharded IDM hot path.

Lanes are independent units (a vehicle reacts only to its leader in the same
lane; no lane changes), so ranks own contiguous whole-lane ranges and never exchange state.
Per optimizer step the only collectives sum the Eq. 4 loss (L = sum_i L_i; 8
bytes) and, in shared-parameter mode, the six parameter gradients (NCCL over NVLink on the GPU
path; gloo in the CPU tests).  The shared gradients travel as per-LANE fp64 rows: each rank
places its own rows (its contiguous lane range) in a zeroed [n_lanes_total, 6] buffer and the
buffer is all-reduced.  Every element has exactly one non-zero contributor, so that all-reduce
is exact (x + 0 + ... + 0 = x in any order): it is an all-gather.  The library then sums the
rows in a fixed order over the global lane index (idm_reduce_shared), so the shared gradient is
bitwise the same for any number of ranks.
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


def world_size(group=None) -> int:
    if not (dist.is_available() and dist.is_initialized()):
        return 1
    return dist.get_world_size(group)


def _all_gather_ints(x: int, group=None) -> list[int]:
    t = torch.tensor([x], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [int(v.item()) for v in out]


def lane_offset(n_lanes_local: int, group=None) -> tuple[int, int]:
    """(first global lane of this rank, total lanes) for contiguous lane shards in rank order."""
    if world_size(group) == 1:
        return 0, n_lanes_local
    sizes = _all_gather_ints(n_lanes_local, group)
    r = dist.get_rank(group)
    return sum(sizes[:r]), sum(sizes)


def sum_over_ranks(x: int, group=None) -> int:
    """Sum of a per-rank integer (e.g. vehicles per rank, for whole-job throughput)."""
    if world_size(group) == 1:
        return x
    return sum(_all_gather_ints(x, group))


def reduce_loss(loss: torch.Tensor, group=None):
    """Sum the Eq. 4 loss (fp64 [1]) over all ranks, in place (8 bytes).  No-op on one rank."""
    if world_size(group) > 1:
        if loss.is_cuda and dist.get_backend(group) == "gloo":
            t = loss.cpu()
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            loss.copy_(t)
        else:
            dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)


reduce_step = reduce_loss  # the per-vehicle-parameter step's only collective


def gather_lane_rows(rows: torch.Tensor, lane0: int, n_lanes_total: int,
                     group=None) -> torch.Tensor:
    """All ranks' per-lane rows [n_lanes_local, w] in global lane order [n_lanes_total, w]:
    this rank's rows at [lane0, lane0 + n_local) of a zeroed buffer, all-reduced.  Exact for
    any reduction order (one non-zero contributor per element)."""
    host = rows.is_cuda and world_size(group) > 1 and dist.get_backend(group) == "gloo"
    dev = torch.device("cpu") if host else rows.device  # gloo reduces host tensors
    buf = torch.zeros(n_lanes_total, rows.shape[1], dtype=rows.dtype, device=dev)
    buf[lane0:lane0 + rows.shape[0]].copy_(rows)
    if world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf.to(rows.device) if host else buf


def reduce_shared_step(sim, lane0: int, n_lanes_total: int, group=None):
    """Shared-parameter mode, between idm_backward and idm_adam_step: gather every rank's
    per-lane gradient rows exactly, sum them in the fixed global lane order in the library
    (idm_reduce_shared -> sim.grad_params) and sum the loss.  One rank: idm_backward already
    reduced the same rows in the same order, so this is a no-op."""
    if world_size(group) == 1:
        return
    buf = gather_lane_rows(sim.lane_grads, lane0, n_lanes_total, group)
    reduce_loss(sim.loss_dev, group)
    sim.reduce_shared(buf)


def max_over_ranks(x: float, device, group=None) -> float:
    """Max of a per-rank scalar (device timing: the slowest rank defines the step)."""
    if not (dist.is_available() and dist.is_initialized()):
        return x
    if dist.get_backend(group) == "gloo":
        device = "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def barrier(group=None):
    """dist.barrier() when distributed, else nothing."""
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group=group)
