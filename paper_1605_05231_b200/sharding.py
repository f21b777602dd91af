"""Multi-GPU plumbing for the view-sharded forward projector.

One process per GPU (torchrun).  Views are independent once the radial lattice
exists, so each rank projects a contiguous view range; ranges are aligned to the
reference's view batches (pipeline.py:105-110) so that no two ranks rebuild the
same per-batch resample grid.  Frames are collected with an all-gather over the
process group (NCCL on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations


def view_batches(n_views: int, per_view: int, target_batch: int) -> list[tuple[int, int]]:
    """pipeline._view_batches (pipeline.py:105-110)."""
    step = max(1, target_batch // per_view)
    return [(lo, min(lo + step, n_views)) for lo in range(0, n_views, step)]


def view_shard(n_views: int, world: int, rank: int, batches=None) -> tuple[int, int]:
    """Contiguous, balanced view range of `rank`; aligned to whole batches when
    `batches` is given and there are at least `world` of them."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if batches and len(batches) >= world:
        nb = len(batches)
        b0, b1 = rank * nb // world, (rank + 1) * nb // world
        return batches[b0][0], batches[b1 - 1][1]
    return rank * n_views // world, (rank + 1) * n_views // world


def gather_views(local, n_views: int, group=None):
    """All-gather per-rank frame blocks (torch tensors, rank order) into the full
    (n_views, nu, nv) stack on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = torch.tensor([local.shape[0]], device=local.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    cap = int(max(int(s.item()) for s in all_sizes))
    buf = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    full = torch.cat([o[: int(s.item())] for o, s in zip(out, all_sizes)])
    if full.shape[0] != n_views:
        raise ValueError("gathered view count does not match the geometry")
    return full


def max_over_ranks(value: float, device="cpu", group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
