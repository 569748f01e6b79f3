"""Filter-index sharding of the multi-channel convolution over GPUs.

PAPER.md §2.3 Fig. 2(c) divides the filters along m and hands each
SM the whole feature map; here the same partition is lifted from SMs to the
GPUs of one box: rank r owns filters [m0, m1), its F slice F[m0:m1] and its O
slice O[m0:m1] are contiguous sub-ranges of the ABI layouts, so a shard is a
plain `conv_multi_ex` call on offset pointers — no repacking and no reduction.
I (<= 803 KB for the BASELINE layers) is broadcast once; O may stay sharded or
be all-gathered (one NCCL all-gather over NVLink/NVSwitch) into the full
O[M][Ho][Wo] layout.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous filter range [m0, m1) of `rank` out of `world`."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(M, world)
    m0 = rank * base + min(rank, extra)
    m1 = m0 + base + (1 if rank < extra else 0)
    return m0, m1


def shard_sizes(M: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_range(M, world, r) for r in range(world))]


def broadcast_input(I: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Replicate I on every rank (once, at setup)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(I, src=src, group=group)
    return I


def sharded_multi(I: torch.Tensor, F: torch.Tensor, precision: str = "fp32", world: int | None = None,
                  rank: int | None = None, out: torch.Tensor | None = None, stream=None):
    """This rank's slice O[m0:m1] of Eq. 1 computed by the CUDA kernels.

    F is the FULL filter tensor [M][C][K][K] (only the rank's contiguous slice
    is read) or already the local slice when world/rank are None."""
    from . import conv
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
    m0, m1 = shard_range(F.shape[0], world, rank)
    Floc = F[m0:m1]
    if Floc.shape[0] == 0:
        C, Wy, Wx = I.shape
        K = F.shape[2]
        return torch.empty((0, Wy - K + 1, Wx - K + 1), device=I.device, dtype=torch.float32)
    return conv.multi(I, Floc.contiguous(), precision, out=out, stream=stream)


def allgather_output(O_local: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """All-gather the filter shards into the full O[M][Ho][Wo] (rank order = m order).

    Equal shards use one all_gather_into_tensor (a single NCCL all-gather);
    unequal shards are padded to the largest and trimmed after."""
    world = dist.get_world_size(group)
    sizes = shard_sizes(M, world)
    Ho, Wo = O_local.shape[1], O_local.shape[2]
    mx = max(sizes)
    send = O_local
    if O_local.shape[0] != mx:
        send = torch.zeros((mx, Ho, Wo), dtype=O_local.dtype, device=O_local.device)
        send[:O_local.shape[0]] = O_local
    buf = torch.empty((world * mx, Ho, Wo), dtype=O_local.dtype, device=O_local.device)
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, send.contiguous(), group=group)
    else:
        dist.all_gather(list(buf.chunk(world)), send.contiguous(), group=group)
    if all(s == mx for s in sizes):
        return buf
    return torch.cat([buf[r * mx: r * mx + sizes[r]] for r in range(world)])
