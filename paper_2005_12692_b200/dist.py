"""Multi-GPU plumbing for batched barcodes.

Images of a batch are independent, so a batch is sharded into contiguous slices, one per rank
(one process per GPU, torch.distributed over NCCL on the GPU box); nothing is exchanged while the
barcodes are computed.  The only collective is the final gather of the variable-length barcodes
onto rank 0 in input order: an all-gather of the per-rank counts, then an all-gather of payloads
padded to the largest count.  Single images are not sharded (replicas only).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [start, stop) of n items for `rank` of `world`."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_barcodes(pairs: torch.Tensor, offsets: torch.Tensor, group=None):
    """Concatenate every rank's (pairs (M,3) int32, offsets (B+1,) int64) in rank order.

    Returns (pairs_all, offsets_all) on every rank (all-gather semantics; rank 0 is the consumer).
    Works with any backend (NCCL for CUDA tensors, gloo for CPU tensors)."""
    world = dist.get_world_size(group)
    dev = pairs.device
    m = torch.tensor([pairs.shape[0], offsets.shape[0] - 1], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(m) for _ in range(world)]
    dist.all_gather(counts, m, group=group)
    counts = [(int(c[0]), int(c[1])) for c in counts]
    mp = max(1, max(c[0] for c in counts))
    mb = max(1, max(c[1] for c in counts))
    pad_p = torch.zeros((mp, 3), dtype=pairs.dtype, device=dev)
    pad_p[: pairs.shape[0]] = pairs
    pad_o = torch.zeros((mb + 1,), dtype=offsets.dtype, device=dev)
    pad_o[: offsets.shape[0]] = offsets
    all_p = [torch.empty_like(pad_p) for _ in range(world)]
    all_o = [torch.empty_like(pad_o) for _ in range(world)]
    dist.all_gather(all_p, pad_p, group=group)
    dist.all_gather(all_o, pad_o, group=group)
    out_p, out_o, base = [], [offsets.new_zeros(1)], 0
    for (npairs, nimg), p, o in zip(counts, all_p, all_o):
        out_p.append(p[:npairs])
        out_o.append(o[1: nimg + 1] + base)
        base += npairs
    return torch.cat(out_p), torch.cat(out_o)
