"""Multi-GPU plumbing: session sharding and the result all-gather.

"this approach still works in multi-GPU environments without additional
operations by evenly distributing the block to GPUs since the hidden layer
calculations for each segment of the CPU memory block are not sequentially
related to each other".  On B200 the independent unit is a whole
session (utterance): its caches and histories live on one GPU, weights are
replicated, and the only cross-device traffic is the all-gather of the
per-query (score, child) results (8 B per query) over NCCL / NVLink.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def session_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous even split; sizes differ by at most one and the first
    ``total % world`` ranks get the larger share."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_results(score: torch.Tensor, child: torch.Tensor) -> torch.Tensor:
    """[n] f32 scores + [n] u32-in-i32 handles -> [n, 2] int32 (score bits, child)."""
    return torch.stack([score.view(torch.int32), child.view(torch.int32)], dim=1)


def unpack_results(packed: torch.Tensor):
    return packed[:, 0].contiguous().view(torch.float32), packed[:, 1].contiguous()


def all_gather_results(score: torch.Tensor, child: torch.Tensor, group=None,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather equal-sized per-rank result blocks -> [world * n, 2] int32,
    rank-major (rank r's block at rows [r*n, (r+1)*n))."""
    world = dist.get_world_size(group)
    mine = pack_results(score, child)
    if out is None:
        out = torch.empty((world * mine.shape[0], 2), dtype=torch.int32, device=mine.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, mine, group=group)
    else:
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, mine, group=group)
        if parts[0].data_ptr() != out.data_ptr():
            torch.cat(parts, out=out)
    return out


def global_order(per_rank_sessions: list[int], B_s: int) -> list[tuple[int, int, int]]:
    """(rank, row_lo, row_hi) blocks in global session-major order for one
    frame: rank r's block holds its sessions' queries, B_s per session."""
    blocks, row = [], 0
    for r, s in enumerate(per_rank_sessions):
        blocks.append((r, row, row + s * B_s))
        row += s * B_s
    return blocks
